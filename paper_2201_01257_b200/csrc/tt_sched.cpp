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
#include <string>
#include <vector>

#include "tt_internal.h"

namespace {

enum OpKind { kSet, kAdd, kContract, kScalar, kCholesky };

struct SchedOp {
  OpKind kind;
  tt_tensor C = nullptr, A = nullptr, B = nullptr;
  std::string cl, al, bl;
  double alpha = 0, beta = 0;
  double* result = nullptr;
  void* ws = nullptr;
  int64_t ws_elems = 0;
  std::vector<tt_tensor> reads, writes;
};

bool has(const std::vector<tt_tensor>& v, tt_tensor t) {
  for (tt_tensor u : v)
    if (u == t) return true;
  return false;
}

bool conflicts(const SchedOp& x, const SchedOp& y) {
  for (tt_tensor w : x.writes)
    if (has(y.writes, w) || has(y.reads, w)) return true;
  for (tt_tensor w : y.writes)
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
    bool ok = cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming) == cudaSuccess;
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
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete s;
  return TT_OK;
}

tt_status tt_sched_set(tt_sched s, tt_tensor C, double alpha) {
  SchedOp op;
  op.kind = kSet;
  op.C = C;
  op.alpha = alpha;
  op.writes = {C};
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
  op.writes = {C};
  op.reads = {A};
  if (beta != 0.0) op.reads.push_back(C);
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
  op.writes = {C};
  op.reads = {A, B};
  if (beta != 0.0) op.reads.push_back(C);
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
  op.writes = {C};
  op.reads = {X, B};
  if (beta != 0.0) op.reads.push_back(C);
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
  op.reads = {A, B};
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

tt_status tt_sched_execute(tt_sched s) {
  if (!s) return set_error(TT_E_ARG, "NULL scheduler");
  tt_ctx ctx = s->ctx;
  if (ctx->device < 0) return set_error(TT_E_STATE, "host-only context cannot execute");
  int64_t n;
  int32_t L;
  std::vector<int32_t> lv(s->ops.size());
  tt_status st = tt_sched_levels(s, lv.data(), &n, &L);
  if (st != TT_OK) return st;
  const cudaStream_t main = ctx->stream;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  const bool concurrent = ctx->nranks == 1 && s->streams.size() > 1;
  for (int32_t l = 0; l < L && st == TT_OK; ++l) {
    std::vector<size_t> ids;
    for (size_t i = 0; i < s->ops.size(); ++i)
      if (lv[i] == l) ids.push_back(i);
    if (!concurrent || ids.size() == 1) {
      for (size_t i : ids)
        if ((st = run_op(ctx, s->ops[i])) != TT_OK) break;
    } else {
      // fork: every stream used by the level waits for the work queued so far on the main stream
      cudaEventRecord(s->fork, main);
      const size_t used = std::min(ids.size(), s->streams.size());
      for (size_t k = 0; k < used; ++k) cudaStreamWaitEvent(s->streams[k], s->fork, 0);
      for (size_t k = 0; k < ids.size() && st == TT_OK; ++k) {
        ctx->stream = s->streams[k % used];
        st = run_op(ctx, s->ops[ids[k]]);
      }
      ctx->stream = main;
      // join: the main stream waits for every stream of the level
      for (size_t k = 0; k < used; ++k) {
        cudaEventRecord(s->done[k], s->streams[k]);
        cudaStreamWaitEvent(main, s->done[k], 0);
      }
    }
    s->levels_executed++;
  }
  ctx->stream = main;
  if (prev >= 0) cudaSetDevice(prev);
  s->ops.clear();
  return st;
}

tt_status tt_sched_stats(tt_sched s, int64_t* queued, int64_t* levels_executed) {
  if (!s) return set_error(TT_E_ARG, "NULL scheduler");
  if (queued) *queued = (int64_t)s->ops.size();
  if (levels_executed) *levels_executed = s->levels_executed;
  return TT_OK;
}

}  // extern "C"
