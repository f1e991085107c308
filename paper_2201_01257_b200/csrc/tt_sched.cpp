// tt_sched.cpp -- the operation scheduler (PAPER §3.2, P178, P191-199, P215).
//
// "The TAMM scheduler employs a data flow analysis over the queued tensor operations ... When two or
// more operations share the same tensor object and one of these operations updates the shared object,
// the operations are marked as conflicting operations that can not be executed in parallel.  This
// operation-graph is used to construct a batch of operations that can be executed in parallel,
// minimizing the total number of global synchronizations" (P215).
//
// Levelization (reading R25, after S464-472): level(op) = 1 + max level of the earlier ops it
// conflicts with (0 if none); a batch is a level.  Read/write sets: set writes C; add / contract /
// Cholesky contraction write C and read C (unless beta == 0), A, B (X); a scalar contraction reads A
// and B.  Execution: the ops of a level run concurrently on the scheduler's CUDA streams (forked from
// the context stream with an event, joined back with one event per stream: one synchronisation point
// per level).  With nranks > 1 the ops of a level run in queue order on the context stream so that
// every rank issues its NCCL calls in the same order (SPMD).
#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>


#include "tt_internal.h"

namespace {

enum OpKind { kSet, kAdd, kContract, kScalar, kCholesky };

// A resource an op reads or writes: a tensor's storage (a view is its root tensor: views share the
// parent's storage, so a view and its parent -- or two views of one parent -- always conflict), or a
// caller workspace byte range (the Cholesky contraction's W batches are written there).
struct Res {
  const void* id;            // root tensor handle, or nullptr for a workspace range
  uintptr_t lo = 0, hi = 0;  // workspace byte range [lo, hi)
};

Res tensor_res(tt_tensor t) {
  while (t && t->view_of) t = t->view_of;
  return {t, 0, 0};
}

Res mem_res(const void* p, int64_t bytes) {
  return {nullptr, (uintptr_t)p, (uintptr_t)p + (uintptr_t)std::max<int64_t>(bytes, 0)};
}

bool same(const Res& a, const Res& b) {
  if (a.id || b.id) return a.id == b.id;
  return a.lo < b.hi && b.lo < a.hi;
}

struct SchedOp {
  OpKind kind;
  tt_tensor C = nullptr, A = nullptr, B = nullptr;
  std::string cl, al, bl;
  double alpha = 0, beta = 0;
  double* result = nullptr;
  void* ws = nullptr;
  int64_t ws_elems = 0;
  std::vector<Res> reads, writes;
};

bool has(const std::vector<Res>& v, const Res& t) {
  for (const Res& u : v)
    if (same(u, t)) return true;
  return false;
}

bool conflicts(const SchedOp& x, const SchedOp& y) {
  for (const Res& w : x.writes)
    if (has(y.writes, w) || has(y.reads, w)) return true;
  for (const Res& w : y.writes)
    if (has(x.reads, w)) return true;
  return false;
}

}  // namespace

struct tt_sched_s {
  tt_ctx ctx = nullptr;
  std::vector<SchedOp> ops;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> done;   // one per stream
  cudaEvent_t fork = nullptr;
  int64_t levels_executed = 0;
  // captured CUDA graph of the queue (tt_sched_capture / tt_sched_replay)
  cudaStream_t cap = nullptr;        // capture stream (the context stream may be the legacy stream)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int32_t graph_levels = 0;
  double* d_results = nullptr;       // device slots of the scalar ops of the graph (in the workspace)
  tt::DevMem mem{true};              // ... their workspace region (long-lived)
  std::vector<std::shared_ptr<void>> held;   // every plan the graph reads: never evicted while it lives
  bool pinned = false;               // counted in ctx->graph_pins (the workspace cannot be re-bound)
  std::vector<double*> h_targets;    // their host destinations
  std::vector<double> h_results;
};

using tt::set_error;

static tt_status push(tt_sched s, SchedOp&& op) {
  if (!s) return set_error(TT_E_ARG, "NULL scheduler");
  s->ops.push_back(std::move(op));
  return TT_OK;
}

extern "C" {

tt_status tt_sched_create(tt_ctx ctx, int32_t nstreams, tt_sched* out) {
  if (!ctx || !out) return set_error(TT_E_ARG, "NULL argument");
  *out = nullptr;
  tt_sched s = new tt_sched_s();
  s->ctx = ctx;
  if (ctx->device >= 0) {
    if (nstreams < 1) nstreams = 1;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    bool ok = cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming) == cudaSuccess &&
              cudaStreamCreateWithFlags(&s->cap, cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; ok && i < nstreams; ++i) {
      cudaStream_t st;
      cudaEvent_t ev;
      ok = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
      if (ok) {
        s->streams.push_back(st);
        s->done.push_back(ev);
      }
    }
    if (prev >= 0) cudaSetDevice(prev);
    if (!ok) {
      tt_sched_destroy(s);
      return set_error(TT_E_CUDA, "cannot create scheduler streams");
    }
  }
  *out = s;
  return TT_OK;
}

tt_status tt_sched_destroy(tt_sched s) {
  if (!s) return TT_OK;
  if (s->ctx && s->ctx->device >= 0) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(s->ctx->device);
    for (cudaStream_t st : s->streams) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
    for (cudaEvent_t e : s->done) cudaEventDestroy(e);
    if (s->fork) cudaEventDestroy(s->fork);
    if (s->cap) cudaStreamDestroy(s->cap);
    if (s->exec) cudaGraphExecDestroy(s->exec);
    if (s->graph) cudaGraphDestroy(s->graph);
    if (prev >= 0) cudaSetDevice(prev);
  }
  if (s->pinned) s->ctx->graph_pins--;
  delete s;
  return TT_OK;
}

tt_status tt_sched_set(tt_sched s, tt_tensor C, double alpha) {
  SchedOp op;
  op.kind = kSet;
  op.C = C;
  op.alpha = alpha;
  op.writes = {tensor_res(C)};
  return push(s, std::move(op));
}

tt_status tt_sched_add(tt_sched s, tt_tensor C, const char* cl, double beta, double alpha, tt_tensor A,
                       const char* al) {
  if (!cl || !al) return set_error(TT_E_ARG, "NULL labels");
  SchedOp op;
  op.kind = kAdd;
  op.C = C;
  op.A = A;
  op.cl = cl;
  op.al = al;
  op.alpha = alpha;
  op.beta = beta;
  op.writes = {tensor_res(C)};
  op.reads = {tensor_res(A)};
  if (beta != 0.0) op.reads.push_back(tensor_res(C));
  return push(s, std::move(op));
}

tt_status tt_sched_contract(tt_sched s, tt_tensor C, const char* cl, double beta, double alpha, tt_tensor A,
                            const char* al, tt_tensor B, const char* bl) {
  if (!cl || !al || !bl) return set_error(TT_E_ARG, "NULL labels");
  SchedOp op;
  op.kind = kContract;
  op.C = C;
  op.A = A;
  op.B = B;
  op.cl = cl;
  op.al = al;
  op.bl = bl;
  op.alpha = alpha;
  op.beta = beta;
  op.writes = {tensor_res(C)};
  op.reads = {tensor_res(A), tensor_res(B)};
  if (beta != 0.0) op.reads.push_back(tensor_res(C));
  return push(s, std::move(op));
}

tt_status tt_sched_contract_cholesky(tt_sched s, tt_tensor C, const char* cl, double beta, double alpha,
                                     tt_tensor X, const char* vl, tt_tensor B, const char* bl, void* workspace,
                                     int64_t ws_elems) {
  if (!cl || !vl || !bl) return set_error(TT_E_ARG, "NULL labels");
  SchedOp op;
  op.kind = kCholesky;
  op.C = C;
  op.A = X;
  op.B = B;
  op.cl = cl;
  op.al = vl;
  op.bl = bl;
  op.alpha = alpha;
  op.beta = beta;
  op.ws = workspace;
  op.ws_elems = ws_elems;
  op.writes = {tensor_res(C), mem_res(workspace, ws_elems * (int64_t)sizeof(double))};
  op.reads = {tensor_res(X), tensor_res(B)};
  if (beta != 0.0) op.reads.push_back(tensor_res(C));
  return push(s, std::move(op));
}

tt_status tt_sched_scalar(tt_sched s, double alpha, tt_tensor A, const char* al, tt_tensor B, const char* bl,
                          double* result) {
  if (!al || !bl || !result) return set_error(TT_E_ARG, "NULL argument");
  SchedOp op;
  op.kind = kScalar;
  op.A = A;
  op.B = B;
  op.al = al;
  op.bl = bl;
  op.alpha = alpha;
  op.result = result;
  op.reads = {tensor_res(A), tensor_res(B)};
  return push(s, std::move(op));
}

tt_status tt_sched_levels(tt_sched s, int32_t* level, int64_t* nops, int32_t* nlevels) {
  if (!s || !nops || !nlevels) return set_error(TT_E_ARG, "NULL argument");
  const size_t n = s->ops.size();
  *nops = (int64_t)n;
  std::vector<int32_t> lv(n, 0);
  int32_t L = 0;
  for (size_t i = 0; i < n; ++i) {
    for (size_t j = 0; j < i; ++j)
      if (conflicts(s->ops[i], s->ops[j]) && lv[j] + 1 > lv[i]) lv[i] = lv[j] + 1;
    L = std::max(L, lv[i] + 1);
  }
  *nlevels = n ? L : 0;
  if (level)
    for (size_t i = 0; i < n; ++i) level[i] = lv[i];
  return TT_OK;
}

static tt_status run_op(tt_ctx ctx, const SchedOp& op) {
  switch (op.kind) {
    case kSet: return tt_set(ctx, op.C, op.alpha);
    case kAdd: return tt_add(ctx, op.C, op.cl.c_str(), op.beta, op.alpha, op.A, op.al.c_str());
    case kContract:
      return tt_contract(ctx, op.C, op.cl.c_str(), op.beta, op.alpha, op.A, op.al.c_str(), op.B, op.bl.c_str());
    case kCholesky:
      return tt_contract_cholesky(ctx, op.C, op.cl.c_str(), op.beta, op.alpha, op.A, op.al.c_str(), op.B,
                                  op.bl.c_str(), op.ws, op.ws_elems);
    case kScalar: return tt_contract_scalar(ctx, op.alpha, op.A, op.al.c_str(), op.B, op.bl.c_str(), op.result);
  }
  return set_error(TT_E_ARG, "unknown op");
}

// runs the queued ops level by level on the context stream (+ the scheduler's streams); in graph mode
// scalar results go to device slots
static tt_status run_levels(tt_sched s, const std::vector<int32_t>& lv, int32_t L, bool graph_mode) {
  tt_ctx ctx = s->ctx;
  const cudaStream_t main = ctx->stream;
  const bool concurrent = ctx->nranks == 1 && s->streams.size() > 1;
  tt_status st = TT_OK;
  std::vector<int> slot(s->ops.size(), -1);
  int ns = 0;
  for (size_t i = 0; i < s->ops.size(); ++i)
    if (s->ops[i].kind == kScalar) slot[i] = ns++;
  auto one = [&](size_t i) {
    ctx->scalar_dev_out = (graph_mode && slot[i] >= 0) ? s->d_results + slot[i] : nullptr;
    tt_status r = run_op(ctx, s->ops[i]);
    ctx->scalar_dev_out = nullptr;
    return r;
  };
  for (int32_t l = 0; l < L && st == TT_OK; ++l) {
    std::vector<size_t> ids;
    for (size_t i = 0; i < s->ops.size(); ++i)
      if (lv[i] == l) ids.push_back(i);
    if (!concurrent || ids.size() == 1) {
      for (size_t i : ids)
        if ((st = one(i)) != TT_OK) break;
    } else {
      // fork: every stream used by the level waits for the work queued so far on the main stream
      cudaEventRecord(s->fork, main);
      const size_t used = std::min(ids.size(), s->streams.size());
      for (size_t k = 0; k < used; ++k) cudaStreamWaitEvent(s->streams[k], s->fork, 0);
      for (size_t k = 0; k < ids.size() && st == TT_OK; ++k) {
        ctx->stream = s->streams[k % used];
        st = one(ids[k]);
      }
      ctx->stream = main;
      // join: the main stream waits for every stream of the level
      for (size_t k = 0; k < used; ++k) {
        cudaEventRecord(s->done[k], s->streams[k]);
        cudaStreamWaitEvent(main, s->done[k], 0);
      }
    }
  }
  ctx->stream = main;
  return st;
}

static void drop_graph(tt_sched s) {
  if (s->exec) cudaGraphExecDestroy(s->exec);
  if (s->graph) cudaGraphDestroy(s->graph);
  s->exec = nullptr;
  s->graph = nullptr;
  s->held.clear();
  s->mem.release();
  s->d_results = nullptr;
  if (s->pinned) s->ctx->graph_pins--;
  s->pinned = false;
}

tt_status tt_sched_execute(tt_sched s) {
  NvtxRange nvtx_("tt_sched_execute");
  if (!s) return set_error(TT_E_ARG, "NULL scheduler");
  tt_ctx ctx = s->ctx;
  if (ctx->device < 0) return set_error(TT_E_STATE, "host-only context cannot execute");
  int64_t n;
  int32_t L;
  std::vector<int32_t> lv(s->ops.size());
  tt_status st = tt_sched_levels(s, lv.data(), &n, &L);
  if (st != TT_OK) return st;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  st = run_levels(s, lv, L, false);
  if (st == TT_OK) s->levels_executed += L;
  if (prev >= 0) cudaSetDevice(prev);
  s->ops.clear();
  drop_graph(s);
  return st;
}

tt_status tt_sched_capture(tt_sched s) {
  NvtxRange nvtx_("tt_sched_capture");
  if (!s) return set_error(TT_E_ARG, "NULL scheduler");
  tt_ctx ctx = s->ctx;
  if (ctx->device < 0) return set_error(TT_E_STATE, "host-only context cannot capture");
  int64_t n;
  int32_t L;
  std::vector<int32_t> lv(s->ops.size());
  tt_status st = tt_sched_levels(s, lv.data(), &n, &L);
  if (st != TT_OK) return st;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  drop_graph(s);
  // 1. build every plan (host work, uploads, device task builders) outside the capture; the
  //    scheduler keeps a reference to each so that none is evicted while the graph reads it
  ctx->prepare_only = true;
  ctx->plan_sink = &s->held;
  for (const SchedOp& op : s->ops)
    if ((st = run_op(ctx, op)) != TT_OK) break;
  ctx->prepare_only = false;
  // 2. device slots for the scalar results (workspace)
  s->h_targets.clear();
  for (const SchedOp& op : s->ops)
    if (op.kind == kScalar) s->h_targets.push_back(op.result);
  s->h_results.assign(s->h_targets.size(), 0.0);
  if (st == TT_OK && !s->h_targets.empty()) {
    void* v = nullptr;
    st = tt::ws_alloc(ctx, s->mem, (int64_t)(s->h_targets.size() * sizeof(double)), &v);
    s->d_results = (double*)v;
  }
  if (st == TT_OK) {
    s->pinned = true;
    ctx->graph_pins++;
  }
  // 3. record the levels into a CUDA graph (profiling events off while capturing)
  if (st == TT_OK) {
    const bool prof = ctx->profiling;
    ctx->profiling = false;
    const cudaStream_t user = ctx->stream;
    ctx->stream = s->cap;          // record on the scheduler's capture stream; replay on the context stream
    cudaError_t e = cudaStreamBeginCapture(s->cap, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) st = set_error(TT_E_CUDA, (std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e)).c_str());
    tt_status rs = TT_OK;
    if (st == TT_OK) rs = run_levels(s, lv, L, true);
    if (st == TT_OK) {
      e = cudaStreamEndCapture(s->cap, &s->graph);
      if (rs != TT_OK) st = rs;
      else if (e != cudaSuccess)
        st = set_error(TT_E_CUDA, (std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e)).c_str());
      else if ((e = cudaGraphInstantiate(&s->exec, s->graph, 0)) != cudaSuccess)
        st = set_error(TT_E_CUDA, (std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e)).c_str());
    }
    ctx->stream = user;
    ctx->profiling = prof;
    s->graph_levels = L;
  }
  ctx->plan_sink = nullptr;
  if (st != TT_OK) drop_graph(s);
  if (prev >= 0) cudaSetDevice(prev);
  return st;
}

tt_status tt_sched_replay(tt_sched s) {
  NvtxRange nvtx_("tt_sched_replay");
  if (!s) return set_error(TT_E_ARG, "NULL scheduler");
  if (!s->exec) return set_error(TT_E_STATE, "no captured graph (call tt_sched_capture)");
  tt_ctx ctx = s->ctx;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  tt_status st = TT_OK;
  cudaError_t e = cudaGraphLaunch(s->exec, ctx->stream);
  ctx->launches += 1;
  if (e != cudaSuccess) st = set_error(TT_E_CUDA, cudaGetErrorString(e));
  if (st == TT_OK && !s->h_targets.empty()) {
    e = cudaMemcpyAsync(s->h_results.data(), s->d_results, s->h_results.size() * sizeof(double),
                        cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) st = set_error(TT_E_CUDA, cudaGetErrorString(e));
    else
      for (size_t i = 0; i < s->h_targets.size(); ++i) *s->h_targets[i] = s->h_results[i];
  }
  if (st == TT_OK) s->levels_executed += s->graph_levels;
  if (prev >= 0) cudaSetDevice(prev);
  return st;
}

tt_status tt_sched_stats(tt_sched s, int64_t* queued, int64_t* levels_executed) {
  if (!s) return set_error(TT_E_ARG, "NULL scheduler");
  if (queued) *queued = (int64_t)s->ops.size();
  if (levels_executed) *levels_executed = s->levels_executed;
  return TT_OK;
}

}  // extern "C"
