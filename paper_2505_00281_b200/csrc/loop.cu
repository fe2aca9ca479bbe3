// loop.cu -- the outer iteration of subspace_iter_eig (ofrr/driver.py:101-111 with the
// time-to-tolerance extension) as ONE CUDA graph with device-side control flow: the
// captured iteration graph runs inside a conditional WHILE node, a one-thread kernel
// decides after every iteration (the host loop's checks, same order and thresholds as
// driver.py EigEngine.run), the FP64 report graph runs inside a conditional IF node and a
// second kernel confirms convergence from its residuals.  No host round trip between
// iterations: the host launches the graph once and reads the control block once.
#include "common.cuh"
#include <algorithm>

namespace ofrr {

static constexpr int LOOP_HIST = 256;
struct LoopCtl {
  int state, it, report_it, pad;
  double prev_est;
  double hist[LOOP_HIST];        // worst leading estimate per iteration
  double hist64[LOOP_HIST];      // worst leading FP64 residual per report (-1: none)
};

// status word layout of driver.py (S_*)
static constexpr int S_MV_FLAGS = 0, S_NKEPT = 1, S_EIG_STATUS = 2, S_NOUT = 3, S_GRAM_FLAGS = 4, S_RESTART = 5;

__global__ void k_loop_init(LoopCtl* c) {
  c->state = 0;
  c->it = 0;
  c->report_it = -1;
  c->prev_est = -1.0;
}

// first: 1 for the first iteration (a report request there goes to the host)
__global__ void k_loop_decide(LoopCtl* c, const int* __restrict__ st, const double* __restrict__ est, int m, int top,
                              int k, double tol, int first, cudaGraphConditionalHandle h_loop,
                              cudaGraphConditionalHandle h_rep) {
  const int it = c->it + 1;
  c->it = it;
  int stop = 0, rep = 0;
  if ((st[S_MV_FLAGS] & 1) || st[S_NKEPT] == 0 || st[S_NKEPT] < k || st[S_GRAM_FLAGS] != 0 ||
      st[S_EIG_STATUS] != 0 || (st[S_RESTART] & 1) || st[S_NOUT] < k) {
    c->state = 3;                       // the host loop re-runs and raises / narrows
    stop = 1;
  } else {
    double worst = 0.0;
    for (int j = 0; j < top; ++j) worst = fmax(worst, est[j]);
    if (!(worst == worst)) worst = INFINITY;
    if (it - 1 < LOOP_HIST) { c->hist[it - 1] = worst; c->hist64[it - 1] = -1.0; }
    const bool stalled = c->prev_est >= 0.0 && worst > 0.5 * c->prev_est && worst < 16.0 * tol;
    c->prev_est = worst;
    const bool last = it >= m;
    if (worst < tol || stalled || last) {
      if (first) { c->state = 3; stop = 1; }
      else rep = 1;
    }
  }
  if (!first) cudaGraphSetConditional(h_rep, rep);     // (the first decision has no IF node:
  cudaGraphSetConditional(h_loop, (stop || rep) ? 0 : 1);   //  an unused handle is invalid)
}

__global__ void k_loop_confirm(LoopCtl* c, const double* __restrict__ res, int m, int top, double tol,
                               cudaGraphConditionalHandle h_loop) {
  const int it = c->it;
  double worst = 0.0;
  for (int j = 0; j < top; ++j) worst = fmax(worst, res[j]);
  if (!(worst == worst)) worst = INFINITY;
  if (it - 1 < LOOP_HIST) c->hist64[it - 1] = worst;
  c->report_it = it;
  int cont = 0;
  if (worst < tol) c->state = 1;
  else if (it >= m) c->state = 2;
  else cont = 1;
  cudaGraphSetConditional(h_loop, cont);
}

// Ladder rung (driver.py EigEngine.run with stop_estimate): the rung is done when its worst
// leading estimate falls below `sw` or stops halving (NaN compares false, as on the host);
// state 4 = done (the host takes the restart block from the last iteration's outputs),
// state 3 = anything else the host loop handles (errors, m exhausted).
__global__ void k_loop_decide_rung(LoopCtl* c, const int* __restrict__ st, const double* __restrict__ est, int m,
                                   int top, int k, double sw, cudaGraphConditionalHandle h_loop) {
  const int it = c->it + 1;
  c->it = it;
  int cont = 0;
  if ((st[S_MV_FLAGS] & 1) || st[S_NKEPT] == 0 || st[S_NKEPT] < k || st[S_GRAM_FLAGS] != 0 ||
      st[S_EIG_STATUS] != 0 || (st[S_RESTART] & 1) || st[S_NOUT] < k) {
    c->state = 3;
  } else {
    double worst = 0.0;
    bool nan = false;
    for (int j = 0; j < top; ++j) {
      const double e = est[j];
      nan |= !(e == e);
      worst = fmax(worst, e);
    }
    if (nan) worst = __longlong_as_double(0x7ff8000000000000ll);   // np.max propagates NaN
    if (it - 1 < LOOP_HIST) { c->hist[it - 1] = worst; c->hist64[it - 1] = -1.0; }
    const bool done = worst < sw || (c->prev_est >= 0.0 && worst > 0.5 * c->prev_est);
    c->prev_est = worst;
    if (it >= m) c->state = 3;
    else if (done) c->state = 4;
    else cont = 1;
  }
  cudaGraphSetConditional(h_loop, cont);
}

size_t loop_ctl_bytes() { return sizeof(LoopCtl); }

#define LOOP_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      ofrr_set_error("loop graph: %s failed: %s", #x, cudaGetErrorString(e_));             \
      return OFRR_ERR_CUDA;                                                                \
    }                                                                                      \
  } while (0)

static int add_kernel(cudaGraphNode_t* out, cudaGraph_t g, const cudaGraphNode_t* deps, size_t nd, void* fn,
                      void** args) {
  cudaKernelNodeParams kp = {};
  kp.func = fn;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(1);
  kp.kernelParams = args;
  LOOP_TRY(cudaGraphAddKernelNode(out, g, deps, nd, &kp));
  return OFRR_OK;
}

int loop_build(cudaGraph_t first, cudaGraph_t steady, cudaGraph_t report, const int* st_first,
               const double* est_first, const int* st_steady, const double* est_steady, const double* res_report,
               const void* copy_src, void* copy_dst, size_t copy_bytes, void* ctl_v, int m, int top, int k,
               double tol, cudaGraphExec_t* exec_out) {
  LoopCtl* ctl = (LoopCtl*)ctl_v;
  cudaGraph_t g;
  LOOP_TRY(cudaGraphCreate(&g, 0));
  int rc = OFRR_OK;
  cudaGraphConditionalHandle h_loop, h_rep;
  cudaGraphNode_t n_init, n_first, n_dec0, n_copy, n_while, prev;
  cudaGraph_t body;
  cudaGraphNodeParams cp = {};
  do {
    if (cudaGraphConditionalHandleCreate(&h_loop, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    {
      void* a[] = {&ctl};
      if ((rc = add_kernel(&n_init, g, nullptr, 0, (void*)k_loop_init, a))) break;
    }
    if (cudaGraphAddChildGraphNode(&n_first, g, &n_init, 1, first) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    // the first iteration's decision: never a report (host), continue -> h_loop = 1
    {
      int one = 1;
      cudaGraphConditionalHandle h_none = 0;
      void* a[] = {&ctl, (void*)&st_first, (void*)&est_first, &m, &top, &k, &tol, &one, &h_loop, &h_none};
      if ((rc = add_kernel(&n_dec0, g, &n_first, 1, (void*)k_loop_decide, a))) break;
    }
    prev = n_dec0;
    if (copy_bytes) {
      if (cudaGraphAddMemcpyNode1D(&n_copy, g, &prev, 1, copy_dst, copy_src, copy_bytes, cudaMemcpyDeviceToDevice) !=
          cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
      prev = n_copy;
    }
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h_loop;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (cudaGraphAddNode(&n_while, g, &prev, 1, &cp) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    body = cp.conditional.phGraph_out[0];
    cudaGraphNode_t b_iter, b_dec, b_if;
    if (cudaGraphAddChildGraphNode(&b_iter, body, nullptr, 0, steady) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    if (cudaGraphConditionalHandleCreate(&h_rep, body, 0, cudaGraphCondAssignDefault) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    {
      int zero = 0;
      void* a[] = {&ctl, (void*)&st_steady, (void*)&est_steady, &m, &top, &k, &tol, &zero, &h_loop, &h_rep};
      if ((rc = add_kernel(&b_dec, body, &b_iter, 1, (void*)k_loop_decide, a))) break;
    }
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = h_rep;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    if (cudaGraphAddNode(&b_if, body, &b_dec, 1, &ip) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    cudaGraph_t rbody = ip.conditional.phGraph_out[0];
    cudaGraphNode_t r_rep, r_conf;
    if (cudaGraphAddChildGraphNode(&r_rep, rbody, nullptr, 0, report) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    {
      void* a[] = {&ctl, (void*)&res_report, &m, &top, &tol, &h_loop};
      if ((rc = add_kernel(&r_conf, rbody, &r_rep, 1, (void*)k_loop_confirm, a))) break;
    }
    cudaError_t e = cudaGraphInstantiate(exec_out, g, 0);
    if (e != cudaSuccess) {
      ofrr_set_error("loop graph: instantiate failed: %s", cudaGetErrorString(e));
      rc = OFRR_ERR_CUDA;
    }
  } while (0);
  if (rc == OFRR_ERR_CUDA) (void)cudaGetLastError();
  cudaGraphDestroy(g);
  return rc;
}

// A ladder rung's loop: first iteration, its decision, then the steady iteration and its
// decision inside a conditional WHILE node (no report).
int loop_build_rung(cudaGraph_t first, cudaGraph_t steady, const int* st_first, const double* est_first,
                    const int* st_steady, const double* est_steady, const void* copy_src, void* copy_dst,
                    size_t copy_bytes, void* ctl_v, int m, int top, int k, double sw, cudaGraphExec_t* exec_out) {
  LoopCtl* ctl = (LoopCtl*)ctl_v;
  cudaGraph_t g;
  LOOP_TRY(cudaGraphCreate(&g, 0));
  int rc = OFRR_OK;
  cudaGraphConditionalHandle h_loop;
  cudaGraphNode_t n_init, n_first, n_dec0, n_copy, n_while, prev;
  cudaGraphNodeParams cp = {};
  do {
    if (cudaGraphConditionalHandleCreate(&h_loop, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    {
      void* a[] = {&ctl};
      if ((rc = add_kernel(&n_init, g, nullptr, 0, (void*)k_loop_init, a))) break;
    }
    if (cudaGraphAddChildGraphNode(&n_first, g, &n_init, 1, first) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    {
      void* a[] = {&ctl, (void*)&st_first, (void*)&est_first, &m, &top, &k, &sw, &h_loop};
      if ((rc = add_kernel(&n_dec0, g, &n_first, 1, (void*)k_loop_decide_rung, a))) break;
    }
    prev = n_dec0;
    if (copy_bytes) {
      if (cudaGraphAddMemcpyNode1D(&n_copy, g, &prev, 1, copy_dst, copy_src, copy_bytes, cudaMemcpyDeviceToDevice) !=
          cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
      prev = n_copy;
    }
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h_loop;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (cudaGraphAddNode(&n_while, g, &prev, 1, &cp) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphNode_t b_iter, b_dec;
    if (cudaGraphAddChildGraphNode(&b_iter, body, nullptr, 0, steady) != cudaSuccess) { rc = OFRR_ERR_CUDA; break; }
    {
      void* a[] = {&ctl, (void*)&st_steady, (void*)&est_steady, &m, &top, &k, &sw, &h_loop};
      if ((rc = add_kernel(&b_dec, body, &b_iter, 1, (void*)k_loop_decide_rung, a))) break;
    }
    cudaError_t e = cudaGraphInstantiate(exec_out, g, 0);
    if (e != cudaSuccess) {
      ofrr_set_error("rung loop graph: instantiate failed: %s", cudaGetErrorString(e));
      rc = OFRR_ERR_CUDA;
    }
  } while (0);
  if (rc == OFRR_ERR_CUDA) (void)cudaGetLastError();
  cudaGraphDestroy(g);
  return rc;
}

}  // namespace ofrr

extern "C" int ofrr_loop_build_rung(void* first_graph, void* steady_graph, const int* st_first,
                                    const double* est_first, const int* st_steady, const double* est_steady,
                                    const void* copy_src, void* copy_dst, size_t copy_bytes, void* ctl, int m, int top,
                                    int k, double sw, void** exec_out) {
  if (!first_graph || !steady_graph || !ctl || !exec_out || m < 1 || top < 1 || top > k) {
    ofrr_set_error("loop_build_rung: invalid arguments");
    return OFRR_ERR_INVALID;
  }
  cudaGraphExec_t ex = nullptr;
  const int rc = ofrr::loop_build_rung((cudaGraph_t)first_graph, (cudaGraph_t)steady_graph, st_first, est_first,
                                       st_steady, est_steady, copy_src, copy_dst, copy_bytes, ctl, m, top, k, sw, &ex);
  *exec_out = (void*)ex;
  return rc;
}

extern "C" size_t ofrr_loop_ctl_bytes(void) { return ofrr::loop_ctl_bytes(); }
extern "C" int ofrr_loop_build(void* first_graph, void* steady_graph, void* report_graph, const int* st_first,
                               const double* est_first, const int* st_steady, const double* est_steady,
                               const double* res_report, const void* copy_src, void* copy_dst, size_t copy_bytes,
                               void* ctl, int m, int top, int k, double tol, void** exec_out) {
  if (!first_graph || !steady_graph || !report_graph || !ctl || !exec_out || m < 1 || top < 1 || top > k) {
    ofrr_set_error("loop_build: invalid arguments");
    return OFRR_ERR_INVALID;
  }
  cudaGraphExec_t ex = nullptr;
  const int rc = ofrr::loop_build((cudaGraph_t)first_graph, (cudaGraph_t)steady_graph, (cudaGraph_t)report_graph,
                                  st_first, est_first, st_steady, est_steady, res_report, copy_src, copy_dst, copy_bytes,
                                  ctl, m, top, k, tol, &ex);
  *exec_out = (void*)ex;
  return rc;
}
extern "C" int ofrr_loop_launch(void* exec, void* stream) {
  const cudaError_t e = cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream);
  if (e != cudaSuccess) { ofrr_set_error("loop_launch: %s", cudaGetErrorString(e)); return OFRR_ERR_CUDA; }
  return OFRR_OK;
}
extern "C" int ofrr_loop_destroy(void* exec) {
  if (exec) cudaGraphExecDestroy((cudaGraphExec_t)exec);
  return OFRR_OK;
}
