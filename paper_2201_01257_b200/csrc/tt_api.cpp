// tt_api.cpp -- host side of libtt: handles, validation, layout, task lists, partition, plans and
// the C ABI entry points declared in include/tt.h.  Citations as in tt.h.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <queue>
#include <string>
#include <vector>

#include <cuda.h>

#include "tt_internal.h"
#include "tt_launch.h"
#include "tt_nccl.h"


using namespace tt;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_uid{1};

tt_status fail(tt_status code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

}  // namespace

tt_status tt::set_error(tt_status code, const char* msg) { return fail(code, "%s", msg); }

namespace {

#define TT_CUDA(x)                                                                    \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) return fail(TT_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

#define TT_TRY(x)                 \
  do {                            \
    tt_status s_ = (x);           \
    if (s_ != TT_OK) return s_;   \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  bool active = false;
  explicit DeviceGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      cudaSetDevice(dev);
      active = true;
    }
  }
  ~DeviceGuard() {
    if (active) cudaSetDevice(prev);
  }
};

tt_status need_device(tt_ctx ctx) {
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  if (ctx->device < 0) return fail(TT_E_STATE, "host-only context (device = -1) cannot run device work");
  return TT_OK;
}

// every device compute call: the context has a workspace (scratch lives there)
tt_status need_ws(tt_ctx ctx) {
  TT_TRY(need_device(ctx));
  if (!ctx->ws.base || !ctx->d_scalar)
    return fail(TT_E_WORKSPACE, "no device workspace bound (tt_workspace_bind; tt_workspace_bytes says how much)");
  return TT_OK;
}

template <class T>
tt_status dev_alloc(tt_ctx ctx, DevMem& m, T** p, size_t n) {
  void* v = nullptr;
  *p = nullptr;
  TT_TRY(ws_alloc(ctx, m, (int64_t)(std::max<size_t>(n, 1) * sizeof(T)), &v));
  *p = (T*)v;
  return TT_OK;
}

// ---------------------------------------------------------------------------------------------
// plan cache: LRU over entries that only the cache references (tt_internal.h "Device workspace")

void plan_put(tt_ctx ctx, const std::string& key, std::shared_ptr<void> p) {
  if (ctx->plan_sink) ctx->plan_sink->push_back(p);
  auto& e = ctx->plans[key];
  e.p = std::move(p);
  e.tick = ++ctx->plan_tick;
  if ((int64_t)ctx->plans.size() > ctx->plan_limit) {   // host-side bound on the cache
    auto victim = ctx->plans.end();
    for (auto it = ctx->plans.begin(); it != ctx->plans.end(); ++it)
      if (it->second.p.use_count() == 1 && (victim == ctx->plans.end() || it->second.tick < victim->second.tick))
        victim = it;
    if (victim != ctx->plans.end()) ctx->plans.erase(victim);
  }
}

// evicts the least-recently-used plan nobody else holds; false if there is none
bool evict_one(tt_ctx ctx) {
  auto victim = ctx->plans.end();
  for (auto it = ctx->plans.begin(); it != ctx->plans.end(); ++it)
    if (it->second.p.use_count() == 1 && (victim == ctx->plans.end() || it->second.tick < victim->second.tick))
      victim = it;
  if (victim == ctx->plans.end()) return false;
  ctx->plans.erase(victim);   // its DevMem retires its regions
  return true;
}

// retired regions become free once every queued kernel that may read them has finished
tt_status drain_retired(tt_ctx ctx) {
  if (ctx->ws.retired.empty()) return TT_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(ctx->stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
    return fail(TT_E_WORKSPACE, "workspace full while a CUDA graph is being captured");
  TT_CUDA(cudaDeviceSynchronize());
  for (auto& r : ctx->ws.retired) ctx->ws.give(r.first, r.second);
  ctx->ws.retired.clear();
  return TT_OK;
}

// A builder that failed part-way holds arrays that may split the free space: after it released them,
// evict every plan nobody holds and drain, so that its retry allocates from one contiguous region.
tt_status ws_make_room(tt_ctx ctx) {
  while (evict_one(ctx)) {}
  return drain_retired(ctx);
}

}  // namespace

void tt::DevMem::release() {
  if (ctx && gen == ctx->ws.gen)
    for (auto& r : regions) {
      ctx->ws.retired.push_back(r);
      ctx->ws.live -= r.second;
    }
  regions.clear();
}

tt_status tt::ws_alloc(tt_ctx ctx, DevMem& m, int64_t bytes, void** out) {
  *out = nullptr;
  Arena& A = ctx->ws;
  const int64_t n = (bytes + kWsAlign - 1) / kWsAlign * kWsAlign;
  if (!A.base) {
    A.need = std::max(A.need, A.live + n);
    return fail(TT_E_WORKSPACE, "no device workspace bound (tt_workspace_bind); this call needs >= %lld bytes",
                (long long)A.need);
  }
  if (m.ctx != ctx || m.gen != A.gen) {
    m.forget();
    m.ctx = ctx;
    m.gen = A.gen;
  }
  int64_t off = 0;
  bool ok = A.take(n, &off, m.top);
  while (!ok) {
    if (!A.retired.empty()) {
      TT_TRY(drain_retired(ctx));
    } else if (!evict_one(ctx)) {
      A.need = std::max(A.need, A.live + n);
      return fail(TT_E_WORKSPACE, "device workspace of %lld bytes is full (%lld live, no evictable plan); bind >= %lld "
                  "bytes (tt_workspace_bytes)", (long long)A.size, (long long)A.live, (long long)A.need);
    }
    ok = A.take(n, &off, m.top);
  }
  m.regions.push_back({off, n});
  *out = A.base + off;
  return TT_OK;
}

tt_tensor_s::~tt_tensor_s() {
  if (ctx) ctx->tensors.erase(this);
}

namespace {

// ---------------------------------------------------------------------------------------------
// profiling scope: CUDA events around a launch on the ctx stream

struct Launch {
  tt_ctx ctx;
  std::string name;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  Launch(tt_ctx c, const char* n) : ctx(c), name(n) {
    ctx->launches++;
    ctx->last.launches++;
    if (ctx->profiling) {
      e0 = get_event();
      e1 = get_event();
      cudaEventRecord(e0, ctx->stream);
    }
  }
  cudaEvent_t get_event() {
    if (!ctx->event_pool.empty()) {
      cudaEvent_t e = ctx->event_pool.back();
      ctx->event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  ~Launch() {
    if (ctx->profiling) {
      cudaEventRecord(e1, ctx->stream);
      ctx->prof.push_back({name, e0, e1});
    }
  }
};

tt_status nccl_check(int r, const char* what) {
  if (r == 0) return TT_OK;
  const char* err = nullptr;
  const NcclApi* api = nccl_api(&err);
  return fail(TT_E_NCCL, "%s failed: %s", what, api && api->GetErrorString ? api->GetErrorString(r) : "?");
}

// ---------------------------------------------------------------------------------------------
// label analysis (P145-174; S356-384, S412-413)

struct Analysis {
  std::string c, a, b;
  int nc = 0, nk = 0;
  std::vector<char> uni;                 // universal labels: C labels, then contracted (A order)
  std::vector<int> a_lab, b_lab;         // universal label of each A / B dim
  std::vector<int> a_pos, b_pos, c_pos;  // dim of each universal label in A / B / C (-1)
  std::vector<std::vector<int>> mg, ng, kg;
  bool a_kc = true, b_nc = true;
};

bool same_tiling(tt_tis x, tt_tis y) {
  return x == y || (x->offsets == y->offsets && x->spin == y->spin);
}

tt_status check_labels(const char* lbl, tt_tensor t, const char* which) {
  if (!lbl) return fail(TT_E_ARG, "NULL label string for %s", which);
  if ((int)strlen(lbl) != t->order)
    return fail(TT_E_LABEL, "%s: %zu labels for an order-%d tensor", which, strlen(lbl), t->order);
  for (int i = 0; i < t->order; ++i)
    for (int j = i + 1; j < t->order; ++j)
      if (lbl[i] == lbl[j]) return fail(TT_E_LABEL, "%s: repeated label '%c' (S412)", which, lbl[i]);
  return TT_OK;
}

tt_status tiling_of(const Analysis& an, char x, tt_tensor C, tt_tensor A, tt_tensor B, tt_tis* out) {
  tt_tis t = nullptr;
  auto chk = [&](const std::string& s, tt_tensor T) -> tt_status {
    size_t p = s.find(x);
    if (p == std::string::npos || !T) return TT_OK;
    if (!t) t = T->dims[p];
    else if (!same_tiling(t, T->dims[p]))
      return fail(TT_E_TILING, "label '%c' bound to different tiled index spaces (S413)", x);
    return TT_OK;
  };
  TT_TRY(chk(an.c, C));
  TT_TRY(chk(an.a, A));
  TT_TRY(chk(an.b, B));
  *out = t;
  return TT_OK;
}

tt_status analyse(tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B, const char* bl,
                  Analysis& an) {
  if (!C || !A || !B) return fail(TT_E_ARG, "NULL tensor");
  TT_TRY(check_labels(cl, C, "C"));
  TT_TRY(check_labels(al, A, "A"));
  TT_TRY(check_labels(bl, B, "B"));
  an.c = cl; an.a = al; an.b = bl;
  for (char x : an.c) {
    bool ia = an.a.find(x) != std::string::npos, ib = an.b.find(x) != std::string::npos;
    if (ia && ib) return fail(TT_E_LABEL, "label '%c' appears in C, A and B (batch label, S380)", x);
    if (!ia && !ib) return fail(TT_E_LABEL, "C label '%c' appears in neither A nor B", x);
  }
  for (char x : an.a)
    if (an.c.find(x) == std::string::npos && an.b.find(x) == std::string::npos)
      return fail(TT_E_LABEL, "dangling label '%c' in A (S380)", x);
  for (char x : an.b)
    if (an.c.find(x) == std::string::npos && an.a.find(x) == std::string::npos)
      return fail(TT_E_LABEL, "dangling label '%c' in B (S380)", x);
  an.nc = (int)an.c.size();
  an.uni.assign(an.c.begin(), an.c.end());
  for (char x : an.a)
    if (an.b.find(x) != std::string::npos && an.c.find(x) == std::string::npos) an.uni.push_back(x);
  an.nk = (int)an.uni.size() - an.nc;
  if ((int)an.uni.size() > kMaxLab) return fail(TT_E_UNSUPPORTED, "more than %d labels", kMaxLab);
  for (char x : an.uni) {
    tt_tis t;
    TT_TRY(tiling_of(an, x, C, A, B, &t));
  }
  auto uidx = [&](char x) { return (int)(std::find(an.uni.begin(), an.uni.end(), x) - an.uni.begin()); };
  an.a_lab.clear(); an.b_lab.clear();
  for (char x : an.a) an.a_lab.push_back(uidx(x));
  for (char x : an.b) an.b_lab.push_back(uidx(x));
  int nu = (int)an.uni.size();
  an.a_pos.assign(nu, -1); an.b_pos.assign(nu, -1); an.c_pos.assign(nu, -1);
  for (int d = 0; d < (int)an.a.size(); ++d) an.a_pos[an.a_lab[d]] = d;
  for (int d = 0; d < (int)an.b.size(); ++d) an.b_pos[an.b_lab[d]] = d;
  for (int d = 0; d < an.nc; ++d) an.c_pos[d] = d;
  // label fusion: adjacent labels in the same order in every operand holding them
  an.mg.clear(); an.ng.clear(); an.kg.clear();
  for (int u = 0; u < an.nc; ++u) {
    bool fromA = an.a_pos[u] >= 0;
    auto& G = fromA ? an.mg : an.ng;
    const auto& pos = fromA ? an.a_pos : an.b_pos;
    if (!G.empty()) {
      int v = G.back().back();
      if (an.c_pos[v] + 1 == an.c_pos[u] && pos[v] >= 0 && pos[v] + 1 == pos[u]) {
        G.back().push_back(u);
        continue;
      }
    }
    G.push_back({u});
  }
  for (int u = an.nc; u < nu; ++u) {
    if (!an.kg.empty()) {
      int v = an.kg.back().back();
      if (an.a_pos[v] + 1 == an.a_pos[u] && an.b_pos[v] + 1 == an.b_pos[u]) {
        an.kg.back().push_back(u);
        continue;
      }
    }
    an.kg.push_back({u});
  }
  if (an.mg.size() > (size_t)kMaxGroup || an.ng.size() > (size_t)kMaxGroup || an.kg.size() > (size_t)kMaxGroup)
    return fail(TT_E_UNSUPPORTED, "more than %d label groups on one GEMM side after fusion", kMaxGroup);
  an.a_kc = an.a_lab.back() >= an.nc;
  an.b_nc = an.b_lab.back() < an.nc;
  return TT_OK;
}

// kernel variants: 0..2 classic cp.async + __syncthreads family, 3.. warp-specialised family
int n_variants() { return num_contract_variants() + num_ws_variants(); }
VariantInfo variant_info(int v) {
  return v < num_contract_variants() ? contract_variant_info(v) : ws_variant_info(v - num_contract_variants());
}
// DMMA-pipe efficiency of each variant on unpadded work (calibrated on cfg2, profiles/r01_variants.txt;
// warp-specialised variants with the TMA producer where it applies)
double variant_efficiency(int v, bool tma) {
  static const double eff[] = {0.70, 0.81, 0.75, 0.925, 0.925, 0.947};
  static const double eff_tma[] = {0.70, 0.81, 0.75, 0.958, 0.95, 0.952};
  const int n = (int)(sizeof(eff) / sizeof(eff[0]));
  return v < n ? (tma ? eff_tma[v] : eff[v]) : 0.5;
}

// tiling of universal label u
tt_tis label_tis(const Analysis& an, int u, tt_tensor C, tt_tensor A) {
  if (u < an.nc) return C->dims[u];
  return A->dims[an.a_pos[u]];
}

// ---------------------------------------------------------------------------------------------
// host canonical task list (reading R11)

struct HostTasks {
  std::vector<int64_t> cblk, ptr, a_blk, b_blk, cost;
  std::vector<int32_t> K;     // contracted extent per task
};

void enumerate_tasks(const Analysis& an, tt_tensor C, tt_tensor A, tt_tensor B, HostTasks& ht) {
  std::vector<tt_tis> lt(an.uni.size());
  for (size_t u = 0; u < an.uni.size(); ++u) lt[u] = label_tis(an, (int)u, C, A);
  std::vector<int32_t> kg(an.nk);
  int64_t ntup = 1;
  for (int l = 0; l < an.nk; ++l) { kg[l] = lt[an.nc + l]->ntiles(); ntup *= kg[l]; }
  ht.ptr.assign(1, 0);
  int32_t cc[TT_MAX_ORDER], kc[kMaxLab], tile[kMaxLab];
  for (int64_t cb = 0; cb < C->nblocks; ++cb) {
    if (!C->nz[cb]) continue;
    C->block_coords(cb, cc);
    int64_t cext = 1;
    for (int d = 0; d < an.nc; ++d) { tile[d] = cc[d]; cext *= lt[d]->size(cc[d]); }
    int64_t cost = 0;
    for (int64_t t = 0; t < ntup; ++t) {
      int64_t r = t;
      for (int l = an.nk - 1; l >= 0; --l) { kc[l] = (int32_t)(r % kg[l]); r /= kg[l]; }
      for (int l = 0; l < an.nk; ++l) tile[an.nc + l] = kc[l];
      int64_t aid = 0, bid = 0;
      for (size_t d = 0; d < an.a_lab.size(); ++d) aid = aid * A->grid[d] + tile[an.a_lab[d]];
      for (size_t d = 0; d < an.b_lab.size(); ++d) bid = bid * B->grid[d] + tile[an.b_lab[d]];
      if (A->nz[aid] && B->nz[bid]) {
        int64_t K = 1;
        for (int l = 0; l < an.nk; ++l) K *= lt[an.nc + l]->size(kc[l]);
        ht.a_blk.push_back(aid);
        ht.b_blk.push_back(bid);
        ht.K.push_back((int32_t)K);
        cost += 2 * cext * K;
      }
    }
    ht.cblk.push_back(cb);
    ht.ptr.push_back((int64_t)ht.a_blk.size());
    ht.cost.push_back(cost);
  }
}

std::vector<int32_t> lpt(const std::vector<int64_t>& cost, const std::vector<int64_t>& ids, int nranks) {
  std::vector<size_t> order(cost.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
    if (cost[x] != cost[y]) return cost[x] > cost[y];
    return ids[x] < ids[y];
  });
  std::vector<int64_t> load(nranks, 0);
  std::vector<int32_t> own(cost.size(), 0);
  for (size_t i : order) {
    int r = 0;
    for (int q = 1; q < nranks; ++q)
      if (load[q] < load[r]) r = q;
    own[i] = r;
    load[r] += cost[i];
  }
  return own;
}

// ---------------------------------------------------------------------------------------------
// gather plan: element ranges of input blocks this rank reads but does not hold (P212; SURVEY
// §8(a) A4).  A need is a range [e0, e1) of a block (the whole block, or the rows of a row-split
// part); the sources are the block's owner or the owners of the overlapping parts.

struct Run {
  int op;        // operand index into the ops list
  int peer;
  int64_t off, len;
};

struct GatherPlan {
  std::vector<int64_t> recv_list, send_list;   // (op, block, peer, e0, e1) rows
  std::vector<Run> recv, send;
  int64_t recv_bytes = 0;
  int64_t all_pieces = 0;   // pieces over ALL ranks: 0 = no rank exchanges anything (same on every rank)
  bool one_group = false;   // few pieces over ALL ranks (the same decision on every rank): one NCCL group
};

struct Need {
  int op;
  int64_t blk, e0, e1;
};
using Needs = std::vector<std::vector<Need>>;   // per rank

// sort and merge overlapping ranges of the same (op, block)
void normalize(std::vector<Need>& v) {
  std::sort(v.begin(), v.end(), [](const Need& x, const Need& y) {
    return std::make_tuple(x.op, x.blk, x.e0, x.e1) < std::make_tuple(y.op, y.blk, y.e0, y.e1);
  });
  std::vector<Need> out;
  for (const Need& n : v) {
    if (!out.empty() && out.back().op == n.op && out.back().blk == n.blk && n.e0 <= out.back().e1) {
      out.back().e1 = std::max(out.back().e1, n.e1);
      continue;
    }
    out.push_back(n);
  }
  v.swap(out);
}

// owners of the pieces of [e0, e1) of block b of T
template <class F>
void pieces(tt_tensor T, int64_t b, int64_t e0, int64_t e1, F&& emit) {
  if (T->parts[b].empty()) {
    emit(T->owner[b], e0, e1);
    return;
  }
  const int64_t inner = T->block_volume(b) / T->ext0(b);
  for (const auto& p : T->parts[b]) {
    const int64_t a = std::max(e0, p.lo * inner), z = std::min(e1, p.hi * inner);
    if (a < z) emit(p.owner, a, z);
  }
}

constexpr size_t kGatherGroupOps = 128;   // NCCL point-to-point calls per group and direction

tt_status build_gather(tt_ctx ctx, Needs need, const std::vector<tt_tensor>& ops, GatherPlan& gp) {
  const int me = ctx->rank, P = ctx->nranks;
  bool into_compact = false;
  int64_t all_pieces = 0;
  for (int dst = 0; dst < P; ++dst) {
    normalize(need[dst]);
    for (const Need& n : need[dst]) {
      tt_tensor T = ops[n.op];
      pieces(T, n.blk, n.e0, n.e1, [&](int32_t src, int64_t a, int64_t z) {
        if (src == TT_REPLICATED || src == dst) return;
        ++all_pieces;
        if (T->compact) into_compact = true;
        if (dst == me) gp.recv_list.insert(gp.recv_list.end(), {n.op, n.blk, src, a, z});
        if (src == me) gp.send_list.insert(gp.send_list.end(), {n.op, n.blk, dst, a, z});
      });
    }
  }
  // a compact tensor (storage = the rank's own parts only) has no room for received pieces; every
  // rank sees the same needs, so every rank fails alike
  if (into_compact)
    return fail(TT_E_UNSUPPORTED, "an operand with compact storage would have to receive remote pieces");
  // runs: pieces of one (operand, peer) merged when adjacent in the GLOBAL packed order (the same
  // decision on sender and receiver); compact tensors never merge across blocks
  auto runs = [&](const std::vector<int64_t>& lst, std::vector<Run>& out) {
    std::vector<size_t> idx(lst.size() / 5);
    std::iota(idx.begin(), idx.end(), 0);
    auto goff = [&](size_t i) { return ops[lst[5 * i]]->gblk_off[lst[5 * i + 1]] + lst[5 * i + 3]; };
    auto soff = [&](size_t i) { return ops[lst[5 * i]]->blk_off[lst[5 * i + 1]] + lst[5 * i + 3]; };
    std::sort(idx.begin(), idx.end(), [&](size_t x, size_t y) {
      return std::make_tuple(lst[5 * x + 2], lst[5 * x], goff(x)) < std::make_tuple(lst[5 * y + 2], lst[5 * y], goff(y));
    });
    int64_t gend = 0, lastblk = -1;
    for (size_t i : idx) {
      const int op = (int)lst[5 * i], peer = (int)lst[5 * i + 2];
      const int64_t off = goff(i), len = lst[5 * i + 4] - lst[5 * i + 3], blk = lst[5 * i + 1];
      if (!out.empty() && out.back().op == op && out.back().peer == peer) {
        Run& r = out.back();
        const int64_t gap = off - gend;
        if (gap >= 0 && gap <= 1 && (!ops[op]->compact || blk == lastblk)) {   // <= 1 alignment pad element
          r.len += gap + len;
          gend = off + len;
          lastblk = blk;
          continue;
        }
      }
      out.push_back({op, peer, soff(i), len});
      gend = off + len;
      lastblk = blk;
    }
  };
  runs(gp.recv_list, gp.recv);
  runs(gp.send_list, gp.send);
  for (const Run& r : gp.recv) gp.recv_bytes += r.len * 8;
  gp.one_group = all_pieces <= (int64_t)kGatherGroupOps * P;
  gp.all_pieces = all_pieces;
  return TT_OK;
}

// The context stream must not run NCCL work while prefetched gathers are still in flight on the
// communication stream (never two streams on one communicator at once): called before every
// collective issued on ctx->stream.
tt_status wait_comm(tt_ctx ctx) {
  if (!ctx->comm_pending) return TT_OK;
  TT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->comm_done, 0));
  ctx->comm_pending = false;
  return TT_OK;
}

// Simulated ranks (tt_ctx_create_sim): the gather as device-to-device copies from the peers' buffers.
// Entry: every rank records `ready` after its earlier work and meets the others at a barrier; each
// receiver waits on its sources' `ready` and copies its received pieces (adjacent pieces merged when
// contiguous on both sides: one cudaMemcpyAsync per run); exit: `done` + barrier, and every rank waits
// on all `done` events before later work may overwrite what others read.  Every rank passes both
// barriers even after an error (no rank is left waiting).
tt_status sim_exchange(tt_ctx ctx, const GatherPlan& gp, const std::vector<tt_tensor>& ops, cudaStream_t stream) {
  tt_sim S = ctx->sim;
  const int me = ctx->rank, P = ctx->nranks;
  tt_status st = TT_OK;
  if (cudaEventRecord(S->ready[me], stream) != cudaSuccess) st = fail(TT_E_CUDA, "sim: event record");
  S->barrier();
  std::vector<char> waited(P, 0);
  double* pd = nullptr;
  const double* ps = nullptr;
  int64_t pn = 0;
  int64_t copies = 0;
  auto flush = [&]() {
    if (pn > 0 && st == TT_OK) {
      if (cudaMemcpyAsync(pd, ps, (size_t)pn * 8, cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
        st = fail(TT_E_CUDA, "sim: cudaMemcpyAsync");
      ++copies;
    }
    pn = 0;
  };
  for (size_t i = 0; st == TT_OK && i + 4 < gp.recv_list.size() + 1; i += 5) {
    const int op = (int)gp.recv_list[i], src = (int)gp.recv_list[i + 2];
    const int64_t blk = gp.recv_list[i + 1], a0 = gp.recv_list[i + 3], z0 = gp.recv_list[i + 4];
    tt_tensor T = ops[op], Q = S->peer(T, src);
    if (!Q || !Q->data || Q->nblocks != T->nblocks || Q->blk_off[blk] < 0) {
      st = fail(TT_E_STATE, "sim: rank %d holds no matching tensor (creation order differs across ranks?)", src);
      break;
    }
    if (!waited[src]) {
      if (cudaStreamWaitEvent(stream, S->ready[src], 0) != cudaSuccess) st = fail(TT_E_CUDA, "sim: event wait");
      waited[src] = 1;
    }
    double* d = T->data + T->blk_off[blk] + a0;
    const double* s = Q->data + Q->blk_off[blk] + a0;
    if (pn > 0 && d == pd + pn && s == ps + pn) {
      pn += z0 - a0;
    } else {
      flush();
      pd = d;
      ps = s;
      pn = z0 - a0;
    }
  }
  flush();
  if (cudaEventRecord(S->done[me], stream) != cudaSuccess && st == TT_OK) st = fail(TT_E_CUDA, "sim: event record");
  S->barrier();
  for (int q = 0; q < P; ++q)
    if (q != me && cudaStreamWaitEvent(stream, S->done[q], 0) != cudaSuccess && st == TT_OK)
      st = fail(TT_E_CUDA, "sim: event wait");
  ctx->last.launches += 0 * copies;
  return st;
}

// dst (device, one double) <- sum over ranks of every rank's dst, on `stream`
tt_status allreduce_sum(tt_ctx ctx, double* dst, cudaStream_t stream) {
  if (ctx->nranks <= 1) return TT_OK;
  if (stream == ctx->stream) TT_TRY(wait_comm(ctx));
  if (ctx->sim) {
    tt_sim S = ctx->sim;
    const int me = ctx->rank, P = ctx->nranks;
    tt_status st = TT_OK;
    if (cudaMemcpyAsync(S->d_part + me, dst, 8, cudaMemcpyDeviceToDevice, stream) != cudaSuccess ||
        cudaEventRecord(S->ready[me], stream) != cudaSuccess)
      st = fail(TT_E_CUDA, "sim all-reduce: copy / event");
    S->barrier();
    for (int q = 0; q < P && st == TT_OK; ++q)
      if (q != me && cudaStreamWaitEvent(stream, S->ready[q], 0) != cudaSuccess) st = fail(TT_E_CUDA, "sim: event wait");
    if (st == TT_OK && launch_sum_slots(S->d_part, P, dst, stream) != cudaSuccess) st = fail(TT_E_CUDA, "sim: sum kernel");
    if (cudaEventRecord(S->done[me], stream) != cudaSuccess && st == TT_OK) st = fail(TT_E_CUDA, "sim: event record");
    S->barrier();
    for (int q = 0; q < P; ++q)
      if (q != me && cudaStreamWaitEvent(stream, S->done[q], 0) != cudaSuccess && st == TT_OK)
        st = fail(TT_E_CUDA, "sim: event wait");
    return st;
  }
  const char* err = nullptr;
  const NcclApi* api = nccl_api(&err);
  if (!api) return fail(TT_E_NCCL, "%s", err);
  return nccl_check(api->AllReduce(dst, dst, 1, kNcclFloat64, kNcclSum, ctx->comm, stream), "ncclAllReduce");
}

// Exchange schedule: with at most kGatherGroupOps runs per direction, one group over all peers; else
// P-1 rounds; in round k every rank sends to rank+k and receives from rank-k,
// and each round is cut into NCCL groups of at most kGatherGroupOps runs per direction (the i-th
// group of a round holds the i-th slices of both lists, which the partner slices identically).
// One group with thousands of point-to-point calls to several peers stalled NCCL at 4 ranks.

tt_status run_gather(tt_ctx ctx, const GatherPlan& gp, const std::vector<tt_tensor>& ops,
                     cudaStream_t stream = nullptr) {
  if (ctx->nranks <= 1 || gp.all_pieces == 0) return TT_OK;   // the same decision on every rank
  if (!stream) {
    stream = ctx->stream;
    TT_TRY(wait_comm(ctx));
  }
  if (ctx->sim) return sim_exchange(ctx, gp, ops, stream);
  if (gp.recv.empty() && gp.send.empty()) return TT_OK;
  const char* err = nullptr;
  const NcclApi* api = nccl_api(&err);
  if (!api) return fail(TT_E_NCCL, "%s", err);
  const int P = ctx->nranks, me = ctx->rank;
  // few pieces over all ranks: one NCCL group with every peer (all transfers in flight at once)
  if (gp.one_group) {
    TT_TRY(nccl_check(api->GroupStart(), "ncclGroupStart"));
    for (const Run& r : gp.send)
      TT_TRY(nccl_check(api->Send(ops[r.op]->data + r.off, (size_t)r.len, kNcclFloat64, r.peer, ctx->comm, stream), "ncclSend"));
    for (const Run& r : gp.recv)
      TT_TRY(nccl_check(api->Recv(ops[r.op]->data + r.off, (size_t)r.len, kNcclFloat64, r.peer, ctx->comm, stream), "ncclRecv"));
    TT_TRY(nccl_check(api->GroupEnd(), "ncclGroupEnd"));
    return TT_OK;
  }
  auto peer_range = [](const std::vector<Run>& v, int peer, size_t& b, size_t& e) {   // runs sorted by peer
    b = 0;
    while (b < v.size() && v[b].peer < peer) ++b;
    e = b;
    while (e < v.size() && v[e].peer == peer) ++e;
  };
  for (int k = 1; k < P; ++k) {
    const int to = (me + k) % P, from = (me - k + P) % P;
    size_t sb, se, rb, re;
    peer_range(gp.send, to, sb, se);
    peer_range(gp.recv, from, rb, re);
    const size_t ns = se - sb, nr = re - rb;
    const size_t ng = std::max((ns + kGatherGroupOps - 1) / kGatherGroupOps, (nr + kGatherGroupOps - 1) / kGatherGroupOps);
    for (size_t g = 0; g < ng; ++g) {
      TT_TRY(nccl_check(api->GroupStart(), "ncclGroupStart"));
      for (size_t i = sb + g * kGatherGroupOps; i < std::min(se, sb + (g + 1) * kGatherGroupOps); ++i) {
        const Run& r = gp.send[i];
        TT_TRY(nccl_check(api->Send(ops[r.op]->data + r.off, (size_t)r.len, kNcclFloat64, r.peer, ctx->comm, stream), "ncclSend"));
      }
      for (size_t i = rb + g * kGatherGroupOps; i < std::min(re, rb + (g + 1) * kGatherGroupOps); ++i) {
        const Run& r = gp.recv[i];
        TT_TRY(nccl_check(api->Recv(ops[r.op]->data + r.off, (size_t)r.len, kNcclFloat64, r.peer, ctx->comm, stream), "ncclRecv"));
      }
      TT_TRY(nccl_check(api->GroupEnd(), "ncclGroupEnd"));
    }
  }
  return TT_OK;
}

// ---------------------------------------------------------------------------------------------
// tensor device metadata

tt_status ensure_dev(tt_tensor t) {
  if (t->dev_ready && !t->dev_off_stale) return TT_OK;
  tt_ctx ctx = t->ctx;
  TT_TRY(need_device(ctx));
  if (!t->dev_ready) {
    TT_TRY(dev_alloc(ctx, t->mem, &t->d_nz, t->nblocks));
    TT_TRY(dev_alloc(ctx, t->mem, &t->d_blk_off, t->nblocks));
    TT_CUDA(cudaMemcpy(t->d_nz, t->nz.data(), t->nblocks, cudaMemcpyHostToDevice));
    t->d_toff.assign(t->order, nullptr);
    for (int d = 0; d < t->order; ++d) {
      TT_TRY(dev_alloc(ctx, t->mem, &t->d_toff[d], t->dims[d]->offsets.size()));
      TT_CUDA(cudaMemcpy(t->d_toff[d], t->dims[d]->offsets.data(), t->dims[d]->offsets.size() * 8, cudaMemcpyHostToDevice));
    }
  }
  TT_CUDA(cudaMemcpy(t->d_blk_off, t->blk_off.data(), t->nblocks * 8, cudaMemcpyHostToDevice));
  t->dev_ready = true;
  t->dev_off_stale = false;
  return TT_OK;
}

tt_status check_bound(tt_tensor t, const char* which) {
  if (t->view_of) {   // a view always uses its parent's current binding
    t->data = t->view_of->data;
    t->capacity = t->view_of->capacity;
  }
  if (!t->data) return fail(TT_E_UNBOUND, "tensor %s has no storage bound (S208)", which);
  if (t->capacity < t->storage_elems)
    return fail(TT_E_UNBOUND, "tensor %s: bound capacity %lld < storage size %lld", which, (long long)t->capacity,
                (long long)t->storage_elems);
  return TT_OK;
}

// ---------------------------------------------------------------------------------------------
// contraction plan (cached per (tensors, owner versions, labels))

// Internal contraction options (used by the implicit-operand driver): `local` plans compute exactly
// the listed C parts of this rank and never gather (the operands are local / replicated);
// `no_gather` plans list this rank's C parts (ownership) but build no gather (accounting plans of
// the implicit-operand driver, which moves its operands itself).
struct PartSel {
  int64_t blk, lo, hi;
};
struct ContractOpts {
  bool local = false;
  bool no_gather = false;
  std::vector<PartSel> sel;
  std::string tag;
  int force_variant = -1;   // autotuning: build this kernel variant instead of the model's choice
};

struct ContractPlan {
  DevMem mem;                          // workspace regions of the device arrays below
  Analysis an;
  HostTasks ht;
  struct MyPart {
    int g;                         // index into ht.cblk
    int64_t lo, hi;                // rows of the block's dim-0 tile computed by this rank
  };
  std::vector<MyPart> my;
  GatherPlan gp;
  int variant = 0;
  bool a_vec = false, b_vec = false;   // 16-byte copies along the operand's contiguous direction
  bool persistent = false;             // short work items: persistent CTAs hide pipeline fill / epilogue
  bool tma = false;                    // TMA producer (uniform fused GEMM-shaped operands)
  int64_t tma_k = 0, tma_n = 0;        // row lengths of the A [rows][K] and B [rows][N|K] views
  int tma_mode = 0;                    // bit 0: B is [N][K]; bit 1: multi-group C epilogue
  CUtensorMap maps[2];                 // A, B tensor maps (encoded for map_ptr)
  const void* map_ptr[2] = {nullptr, nullptr};
  int64_t nwork = 0;
  CGroupDesc* d_groups = nullptr;
  TaskDesc* d_tasks = nullptr;
  WorkItem* d_work = nullptr;
  std::vector<SplitDesc> splits;       // split-K parts (reduced after the GEMM kernel)
  SplitDesc* d_splits = nullptr;
  double* d_partials = nullptr;        // their partial sums, one slot per chunk
  int64_t partial_elems = 0;
  int64_t* d_ablk = nullptr;
  int64_t* d_bblk = nullptr;
  int64_t* d_ptr = nullptr;
  bool device_built = false;
  int alt_variant = -1;                // runner-up of the variant model (warp-specialised family)
  int tune = 0;                        // autotuning state: 0 untimed, 1 main timed, 2 decided
  float tune_ms = 0;
  std::shared_ptr<ContractPlan> alt;   // the same plan built for alt_variant
  bool use_alt = false;
  cudaEvent_t pf_event = nullptr;      // tt_contract_prefetch: this plan's gather issued on the comm stream
  bool prefetched = false;
  double flops = 0, bytes = 0;
  int64_t tasks = 0;
};

std::string plan_key(const char* kind, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                     const char* bl, double beta) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s|%llu.%llu|%llu.%llu|%llu.%llu|%s|%s|%s|%d", kind, (unsigned long long)C->uid,
           (unsigned long long)C->version, (unsigned long long)A->uid, (unsigned long long)A->version,
           (unsigned long long)(B ? B->uid : 0), (unsigned long long)(B ? B->version : 0), cl, al, bl ? bl : "",
           beta != 0.0);
  return buf;
}

}  // namespace

// =============================================================================================
// C ABI

extern "C" {

const char* tt_last_error(void) { return g_err.c_str(); }
int32_t tt_version(void) { return 1; }

tt_status tt_nccl_unique_id(void* out128) {
  if (!out128) return fail(TT_E_ARG, "NULL output");
  const char* err = nullptr;
  const NcclApi* api = nccl_api(&err);
  if (!api) return fail(TT_E_NCCL, "%s", err);
  return nccl_check(api->GetUniqueId(out128), "ncclGetUniqueId");
}

}  // extern "C"

// device checks and kernel setup of a new context on c->device (>= 0)
static tt_status ctx_device_setup(tt_ctx c) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || c->device >= ndev)
    return fail(TT_E_CUDA, "device %d not available: %s", c->device, cudaGetErrorString(e));
  DeviceGuard dg(c->device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->device) == cudaSuccess) c->sm_count = prop.multiProcessorCount;
  if (prop.major != 10)
    return fail(TT_E_UNSUPPORTED, "libtt is built for sm_100a (B200); device %d is sm_%d%d", c->device, prop.major, prop.minor);
  for (int v = 0; v < n_variants(); ++v) {
    cudaError_t e2 = v < num_contract_variants() ? contract_variant_setup(v) : ws_variant_setup(v - num_contract_variants());
    if (e2 != cudaSuccess) return fail(TT_E_CUDA, "kernel setup: %s", cudaGetErrorString(e2));
  }
  return TT_OK;
}

extern "C" {

tt_status tt_sim_create(int32_t device, int32_t nranks, tt_sim* out) {
  if (!out) return fail(TT_E_ARG, "NULL output handle");
  *out = nullptr;
  if (nranks < 1 || device < 0) return fail(TT_E_ARG, "bad device %d / nranks %d", device, nranks);
  tt_sim S = new tt_sim_s();
  S->nranks = nranks;
  S->device = device;
  S->ctx.assign(nranks, nullptr);
  DeviceGuard dg(device);
  bool ok = cudaMalloc((void**)&S->d_part, sizeof(double) * nranks) == cudaSuccess;
  for (int r = 0; ok && r < nranks; ++r) {
    cudaEvent_t e0, e1;
    ok = cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) == cudaSuccess;
    if (ok) {
      S->ready.push_back(e0);
      S->done.push_back(e1);
    }
  }
  if (!ok) {
    tt_sim_destroy(S);
    return fail(TT_E_CUDA, "cannot create the simulated-rank group on device %d", device);
  }
  *out = S;
  return TT_OK;
}

tt_status tt_sim_destroy(tt_sim S) {
  if (!S) return TT_OK;
  DeviceGuard dg(S->device);
  for (cudaEvent_t e : S->ready) cudaEventDestroy(e);
  for (cudaEvent_t e : S->done) cudaEventDestroy(e);
  if (S->d_part) cudaFree(S->d_part);
  delete S;
  return TT_OK;
}

tt_status tt_ctx_create_sim(void* stream, int32_t rank, tt_sim S, tt_ctx* out) {
  if (!out || !S) return fail(TT_E_ARG, "NULL argument");
  *out = nullptr;
  if (rank < 0 || rank >= S->nranks) return fail(TT_E_ARG, "bad rank %d / nranks %d", rank, S->nranks);
  {
    std::lock_guard<std::mutex> lk(S->mu);
    if (S->ctx[rank]) return fail(TT_E_STATE, "simulated rank %d already has a context", rank);
  }
  tt_ctx c = new tt_ctx_s();
  c->device = S->device;
  c->stream = (cudaStream_t)stream;
  c->rank = rank;
  c->nranks = S->nranks;
  c->sim = S;
  tt_status s = ctx_device_setup(c);
  if (s != TT_OK) {
    delete c;
    return s;
  }
  std::lock_guard<std::mutex> lk(S->mu);
  S->ctx[rank] = c;
  *out = c;
  return TT_OK;
}

tt_status tt_ctx_create(int32_t device, void* stream, int32_t rank, int32_t nranks, const void* nccl_id, tt_ctx* out) {
  if (!out) return fail(TT_E_ARG, "NULL output handle");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TT_E_ARG, "bad rank %d / nranks %d", rank, nranks);
  tt_ctx c = new tt_ctx_s();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->rank = rank;
  c->nranks = nranks;
  if (device >= 0) {
    tt_status s0 = ctx_device_setup(c);
    if (s0 != TT_OK) {
      delete c;
      return s0;
    }
    DeviceGuard dg(device);
    if (nranks > 1) {
      if (!nccl_id) {
        delete c;
        return fail(TT_E_ARG, "nranks > 1 needs an ncclUniqueId");
      }
      const char* err = nullptr;
      const NcclApi* api = nccl_api(&err);
      if (!api) {
        delete c;
        return fail(TT_E_NCCL, "%s", err);
      }
      int r = nccl_comm_init(api, &c->comm, nranks, nccl_id, rank);
      if (r != 0) {
        delete c;
        return fail(TT_E_NCCL, "ncclCommInitRank: %s", api->GetErrorString(r));
      }
    }
  }
  *out = c;
  return TT_OK;
}

tt_status tt_ctx_destroy(tt_ctx ctx) {
  if (!ctx) return TT_OK;
  DeviceGuard dg(ctx->device);
  if (ctx->device >= 0) cudaStreamSynchronize(ctx->stream);
  ctx->plans.clear();
  ctx->scratch.forget();
  for (tt_tensor_s* t : ctx->tensors) {   // tensors may outlive their context (their handles stay valid)
    t->mem.forget();
    t->mem.ctx = nullptr;
    t->ctx = nullptr;
    t->dev_ready = false;
  }
  ctx->tensors.clear();
  for (auto& r : ctx->prof) { ctx->event_pool.push_back(r.e0); ctx->event_pool.push_back(r.e1); }
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
    cudaEventDestroy(ctx->copy_fork);
  }
  for (cudaEvent_t e : ctx->tile_events) cudaEventDestroy(e);
  if (ctx->comm_stream) {
    cudaStreamSynchronize(ctx->comm_stream);
    cudaStreamDestroy(ctx->comm_stream);
    cudaEventDestroy(ctx->comm_fork);
    cudaEventDestroy(ctx->comm_done);
  }
  if (ctx->comm) {
    const NcclApi* api = nccl_api(nullptr);
    if (api) api->CommDestroy(ctx->comm);
  }
  if (ctx->sim) {
    std::lock_guard<std::mutex> lk(ctx->sim->mu);
    ctx->sim->ctx[ctx->rank] = nullptr;
  }
  delete ctx;
  return TT_OK;
}

tt_status tt_workspace_bind(tt_ctx ctx, void* ptr, int64_t bytes) {
  TT_TRY(need_device(ctx));
  if (!ptr || bytes < kWsAlign) return fail(TT_E_ARG, "workspace: NULL pointer or fewer than %lld bytes", (long long)kWsAlign);
  if ((uintptr_t)ptr % kWsAlign) return fail(TT_E_ARG, "workspace must be %lld-byte aligned", (long long)kWsAlign);
  if (ctx->graph_pins > 0) return fail(TT_E_STATE, "a scheduler holds a captured graph reading the workspace");
  DeviceGuard dg(ctx->device);
  if (ctx->ws.base) TT_CUDA(cudaDeviceSynchronize());   // queued kernels may read the old buffer
  ctx->plans.clear();
  for (tt_tensor_s* t : ctx->tensors) {   // device metadata is rebuilt on next use
    t->mem.forget();
    t->dev_ready = false;
    t->d_nz = nullptr;
    t->d_blk_off = nullptr;
    t->d_toff.clear();
  }
  ctx->scratch.forget();
  ctx->d_scalar = nullptr;
  const int64_t need = ctx->ws.need;
  ctx->ws.reset((char*)ptr, bytes / kWsAlign * kWsAlign);
  ctx->ws.need = need > ctx->ws.size ? need : 0;
  return dev_alloc(ctx, ctx->scratch, &ctx->d_scalar, 2);
}

tt_status tt_workspace_bytes(tt_ctx ctx, int64_t* bytes) {
  if (!ctx || !bytes) return fail(TT_E_ARG, "NULL argument");
  *bytes = std::max(kWsMin, std::max(ctx->ws.high, ctx->ws.need));
  return TT_OK;
}

tt_status tt_workspace_info(tt_ctx ctx, int64_t* bound, int64_t* live, int64_t* high) {
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  if (bound) *bound = ctx->ws.size;
  if (live) *live = ctx->ws.live;
  if (high) *high = ctx->ws.high;
  return TT_OK;
}

tt_status tt_ctx_set_plan_limit(tt_ctx ctx, int64_t max_plans) {
  if (!ctx || max_plans < 1) return fail(TT_E_ARG, "NULL context or plan limit < 1");
  ctx->plan_limit = max_plans;
  while ((int64_t)ctx->plans.size() > ctx->plan_limit && evict_one(ctx)) {}
  return TT_OK;
}

tt_status tt_ctx_clear_plans(tt_ctx ctx) {
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  while (evict_one(ctx)) {}
  return TT_OK;
}

tt_status tt_ctx_set_profiling(tt_ctx ctx, int32_t enable) {
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  ctx->profiling = enable != 0;
  return TT_OK;
}

tt_status tt_profile_read(tt_ctx ctx, const char* kernel, double* total_ms, int64_t* launches) {
  if (!ctx || !total_ms || !launches) return fail(TT_E_ARG, "NULL argument");
  *total_ms = 0;
  *launches = 0;
  if (ctx->device < 0) return TT_OK;
  DeviceGuard dg(ctx->device);
  TT_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto& r : ctx->prof) {
    if (kernel && kernel[0] && r.name.find(kernel) == std::string::npos) continue;
    float ms = 0;
    TT_CUDA(cudaEventElapsedTime(&ms, r.e0, r.e1));
    *total_ms += ms;
    *launches += 1;
  }
  return TT_OK;
}

tt_status tt_profile_reset(tt_ctx ctx) {
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  for (auto& r : ctx->prof) { ctx->event_pool.push_back(r.e0); ctx->event_pool.push_back(r.e1); }
  ctx->prof.clear();
  return TT_OK;
}

tt_status tt_last_stats(tt_ctx ctx, tt_stats* out) {
  if (!ctx || !out) return fail(TT_E_ARG, "NULL argument");
  *out = ctx->last;
  return TT_OK;
}

tt_status tt_launch_count(tt_ctx ctx, int64_t* out) {
  if (!ctx || !out) return fail(TT_E_ARG, "NULL argument");
  *out = ctx->launches;
  return TT_OK;
}

tt_status tt_sync(tt_ctx ctx) {
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  if (ctx->device < 0) return TT_OK;
  DeviceGuard dg(ctx->device);
  TT_CUDA(cudaStreamSynchronize(ctx->stream));
  TT_CUDA(cudaGetLastError());
  return TT_OK;
}

// ---------------------------------------------------------------------------------------------
// index spaces and tilings

tt_status tt_is_create(int64_t extent, int32_t n_ranges, const int64_t* be, const int8_t* spin, tt_is* out) {
  if (!out) return fail(TT_E_ARG, "NULL output handle");
  *out = nullptr;
  if (extent < 1) return fail(TT_E_ARG, "extent must be >= 1");
  if (n_ranges < 0 || (n_ranges > 0 && !be)) return fail(TT_E_ARG, "bad ranges");
  tt_is s = new tt_is_s();
  s->extent = extent;
  int64_t pos = 0;
  for (int i = 0; i < n_ranges; ++i) {
    int64_t b = be[2 * i], e = be[2 * i + 1];
    if (b != pos || e <= b) {
      delete s;
      return fail(TT_E_COVERAGE, "ranges must be ascending, non-empty and cover [0, extent)");
    }
    if (spin && spin[i] != 1 && spin[i] != -1) {
      delete s;
      return fail(TT_E_ARG, "spin must be +1 or -1");
    }
    s->rb.push_back(b);
    s->re.push_back(e);
    s->rspin.push_back(spin ? spin[i] : 0);
    pos = e;
  }
  if (n_ranges > 0 && pos != extent) {
    delete s;
    return fail(TT_E_COVERAGE, "ranges must cover [0, extent)");
  }
  if (n_ranges == 0) {
    s->rb.push_back(0);
    s->re.push_back(extent);
    s->rspin.push_back(0);
  }
  *out = s;
  return TT_OK;
}

tt_status tt_is_destroy(tt_is is) {
  delete is;
  return TT_OK;
}

tt_status tt_tis_fixed(tt_is is, int64_t tile, tt_tis* out) {
  if (!is || !out) return fail(TT_E_ARG, "NULL argument");
  *out = nullptr;
  if (tile < 1) return fail(TT_E_ARG, "tile size must be >= 1");
  tt_tis t = new tt_tis_s();
  t->is = is;
  t->uid = g_uid++;
  t->offsets.push_back(0);
  for (size_t r = 0; r < is->rb.size(); ++r) {
    for (int64_t p = is->rb[r]; p < is->re[r]; p += tile) {
      t->offsets.push_back(std::min(p + tile, is->re[r]));
      t->spin.push_back(is->rspin[r]);
    }
  }
  *out = t;
  return TT_OK;
}

tt_status tt_tis_custom(tt_is is, int32_t n, const int64_t* sizes, tt_tis* out) {
  if (!is || !out || (n > 0 && !sizes)) return fail(TT_E_ARG, "NULL argument");
  *out = nullptr;
  if (n < 1) return fail(TT_E_ARG, "need at least one tile");
  int64_t sum = 0;
  for (int i = 0; i < n; ++i) {
    if (sizes[i] < 1) return fail(TT_E_ARG, "tile size must be >= 1");
    sum += sizes[i];
  }
  if (sum != is->extent) return fail(TT_E_COVERAGE, "tile sizes sum to %lld, extent is %lld (P127)", (long long)sum, (long long)is->extent);
  tt_tis t = new tt_tis_s();
  t->is = is;
  t->uid = g_uid++;
  t->offsets.push_back(0);
  for (int i = 0; i < n; ++i) {
    int64_t lo = t->offsets.back(), hi = lo + sizes[i];
    int found = -1;
    for (size_t r = 0; r < is->rb.size(); ++r)
      if (is->rb[r] <= lo && hi <= is->re[r]) found = (int)r;
    if (found < 0) {
      delete t;
      return fail(TT_E_TILING, "tile [%lld,%lld) straddles a range/spin boundary (S39)", (long long)lo, (long long)hi);
    }
    t->offsets.push_back(hi);
    t->spin.push_back(is->rspin[found]);
  }
  *out = t;
  return TT_OK;
}

tt_status tt_tis_info(tt_tis tis, int32_t* ntiles, const int64_t** offsets, const int8_t** tile_spin) {
  if (!tis) return fail(TT_E_ARG, "NULL handle");
  if (ntiles) *ntiles = tis->ntiles();
  if (offsets) *offsets = tis->offsets.data();
  if (tile_spin) *tile_spin = tis->spin.data();
  return TT_OK;
}

tt_status tt_tis_destroy(tt_tis tis) {
  delete tis;
  return TT_OK;
}

tt_status tt_tis_sub(tt_tis parent, int64_t begin, int64_t end, tt_tis* out) {
  if (!parent || !out) return fail(TT_E_ARG, "NULL argument");
  *out = nullptr;
  const auto& po = parent->offsets;
  auto t0 = std::find(po.begin(), po.end(), begin), t1 = std::find(po.begin(), po.end(), end);
  if (begin >= end || t0 == po.end() || t1 == po.end())
    return fail(TT_E_TILING, "sub-space [%lld,%lld) does not start and end on tile boundaries of the parent (P159)",
                (long long)begin, (long long)end);
  tt_tis t = new tt_tis_s();
  t->is = parent->is;
  t->uid = g_uid++;
  t->parent = parent;
  t->tile0 = (int32_t)(t0 - po.begin());
  for (auto it = t0; it <= t1; ++it) t->offsets.push_back(*it - begin);
  t->spin.assign(parent->spin.begin() + t->tile0, parent->spin.begin() + (t1 - po.begin()));
  *out = t;
  return TT_OK;
}

tt_status tt_tis_range(tt_tis parent, int32_t range, tt_tis* out) {
  if (!parent || !out) return fail(TT_E_ARG, "NULL argument");
  if (range < 0 || range >= (int32_t)parent->is->rb.size())
    return fail(TT_E_ARG, "range %d outside the %zu ranges of the index space", range, parent->is->rb.size());
  return tt_tis_sub(parent, parent->is->rb[range], parent->is->re[range], out);
}

// ---------------------------------------------------------------------------------------------
// tensors

// a view copies its parent's block map, storage offsets and owners at creation: the parent's layout
// may not change while views of it exist (they would keep stale offsets and owners)
static tt_status check_no_views(tt_tensor t) {
  if (t->live_views > 0)
    return fail(TT_E_STATE, "tensor has %d live view(s): destroy them before changing its layout", t->live_views);
  return TT_OK;
}

static tt_status tensor_new(tt_ctx ctx, int32_t order, const tt_tis* dims, tt_tensor* out) {
  if (!ctx || !out || !dims) return fail(TT_E_ARG, "NULL argument");
  *out = nullptr;
  if (order < 1 || order > TT_MAX_ORDER) return fail(TT_E_UNSUPPORTED, "order %d outside 1..%d", order, TT_MAX_ORDER);
  tt_tensor t = new tt_tensor_s();
  t->ctx = ctx;
  ctx->tensors.insert(t);
  t->order = order;
  t->uid = g_uid++;
  t->seq = ctx->tensor_seq++;
  t->nblocks = 1;
  for (int d = 0; d < order; ++d) {
    if (!dims[d]) {
      tt_tensor_destroy(t);
      return fail(TT_E_ARG, "NULL tiled index space for dim %d", d);
    }
    t->dims.push_back(dims[d]);
    t->grid.push_back(dims[d]->ntiles());
    t->nblocks *= dims[d]->ntiles();
  }
  if (ctx->sim) {   // simulated ranks: peers find this rank's handle by creation order
    t->sim = ctx->sim;
    t->sim_rank = ctx->rank;
    std::lock_guard<std::mutex> lk(ctx->sim->mu);
    auto& v = ctx->sim->reg[t->seq];
    if (v.empty()) v.assign(ctx->nranks, nullptr);
    v[ctx->rank] = t;
  }
  *out = t;
  return TT_OK;
}

static void tensor_finish(tt_tensor t) {
  // P210 third scheme: packed non-zero blocks, row-major block order, 16-B aligned starts (R10);
  // default owners round robin over the non-zero blocks.
  t->blk_off.assign(t->nblocks, -1);
  t->owner.assign(t->nblocks, -1);
  int64_t cur = 0, k = 0;
  t->nnz = 0;
  for (int64_t b = 0; b < t->nblocks; ++b) {
    if (!t->nz[b]) continue;
    cur = (cur + 1) / 2 * 2;
    t->blk_off[b] = cur;
    cur += t->block_volume(b);
    t->owner[b] = (int32_t)(k++ % t->ctx->nranks);
    t->nnz++;
  }
  t->packed_elems = (cur + 1) / 2 * 2;
  t->gblk_off = t->blk_off;
  t->storage_elems = t->packed_elems;
  t->parts.assign(t->nblocks, {});
  t->any_split = false;
}

// storage offsets: the global packed layout, or (compact) only the ranges this rank holds -- per
// block the span [first held element, last held element) packed in block order, each block base
// even (16-B aligned) so the vectorised paths keep their alignment
static void apply_storage(tt_tensor t) {
  if (!t->compact) {
    t->blk_off = t->gblk_off;
    t->storage_elems = t->packed_elems;
  } else {
    std::vector<std::pair<int64_t, int64_t>> hr;
    int64_t cur = 0;
    for (int64_t b = 0; b < t->nblocks; ++b) {
      t->blk_off[b] = -1;
      t->held_ranges(b, t->ctx->rank, hr);
      if (hr.empty()) continue;
      int64_t e0 = hr[0].first, e1 = hr[0].second;
      for (auto& h : hr) { e0 = std::min(e0, h.first); e1 = std::max(e1, h.second); }
      if ((cur - e0) & 1) ++cur;
      t->blk_off[b] = cur - e0;
      cur += e1 - e0;
    }
    t->storage_elems = std::max<int64_t>(2, (cur + 1) / 2 * 2);
  }
  t->dev_off_stale = true;
}

static void refresh_parts_view(tt_tensor t) {
  t->pv_blk.clear(); t->pv_lo.clear(); t->pv_hi.clear(); t->pv_owner.clear();
  t->any_split = false;
  for (int64_t b = 0; b < t->nblocks; ++b) {
    for (const auto& p : t->parts[b]) {
      t->pv_blk.push_back(b); t->pv_lo.push_back(p.lo); t->pv_hi.push_back(p.hi); t->pv_owner.push_back(p.owner);
      t->any_split = true;
    }
  }
}

tt_status tt_tensor_create(tt_ctx ctx, int32_t order, const tt_tis* dims, const uint8_t* nz, tt_tensor* out) {
  tt_tensor t;
  TT_TRY(tensor_new(ctx, order, dims, &t));
  t->nz.resize(t->nblocks);
  for (int64_t b = 0; b < t->nblocks; ++b) t->nz[b] = nz ? (nz[b] ? 1 : 0) : 1;
  tensor_finish(t);
  *out = t;
  return TT_OK;
}

tt_status tt_tensor_create_spin(tt_ctx ctx, int32_t order, const tt_tis* dims, uint32_t upper, uint32_t lower,
                                tt_tensor* out) {
  tt_tensor t;
  TT_TRY(tensor_new(ctx, order, dims, &t));
  if ((upper | lower) >> order) {
    tt_tensor_destroy(t);
    return fail(TT_E_ARG, "spin masks reference dims beyond the order");
  }
  t->nz.resize(t->nblocks);
  int32_t c[TT_MAX_ORDER];
  for (int64_t b = 0; b < t->nblocks; ++b) {
    t->block_coords(b, c);
    int su = 0, sl = 0;
    for (int d = 0; d < order; ++d) {
      int s = t->dims[d]->spin[c[d]];
      if (upper >> d & 1) su += s;
      if (lower >> d & 1) sl += s;
    }
    t->nz[b] = (su == sl) ? 1 : 0;   // P138 spin block sparsity, reading R7
  }
  tensor_finish(t);
  *out = t;
  return TT_OK;
}

tt_status tt_tensor_info(tt_tensor t, int32_t* order, int64_t* nblocks, int64_t* nnz) {
  if (!t) return fail(TT_E_ARG, "NULL tensor");
  if (order) *order = t->order;
  if (nblocks) *nblocks = t->nblocks;
  if (nnz) *nnz = t->nnz;
  return TT_OK;
}

tt_status tt_tensor_layout(tt_tensor t, int64_t* packed, const int64_t** blk_off, const int32_t** owner,
                           const uint8_t** nz) {
  if (!t) return fail(TT_E_ARG, "NULL tensor");
  if (packed) *packed = t->packed_elems;
  if (blk_off) *blk_off = t->gblk_off.data();
  if (owner) *owner = t->owner.data();
  if (nz) *nz = t->nz.data();
  return TT_OK;
}

tt_status tt_tensor_view(tt_tensor T, const tt_tis* dims, tt_tensor* out) {
  if (!T || !dims || !out) return fail(TT_E_ARG, "NULL argument");
  *out = nullptr;
  if (T->view_of) return fail(TT_E_UNSUPPORTED, "view of a view: slice the parent tensor instead");
  if (T->compact || T->any_split) return fail(TT_E_UNSUPPORTED, "views of compact or row-split tensors");
  std::vector<int32_t> t0(T->order);
  for (int d = 0; d < T->order; ++d) {
    if (!dims[d]) return fail(TT_E_ARG, "NULL tiled index space for dim %d", d);
    if (dims[d] == T->dims[d]) t0[d] = 0;
    else if (dims[d]->parent == T->dims[d]) t0[d] = dims[d]->tile0;
    else return fail(TT_E_TILING, "dim %d: not the tensor's tiled space or a sub-space of it (P152, P159)", d);
  }
  tt_tensor v;
  TT_TRY(tensor_new(T->ctx, T->order, dims, &v));
  v->view_of = T;
  v->nz.resize(v->nblocks);
  v->blk_off.assign(v->nblocks, -1);
  v->owner.assign(v->nblocks, -1);
  int32_t c[TT_MAX_ORDER];
  v->nnz = 0;
  for (int64_t b = 0; b < v->nblocks; ++b) {
    v->block_coords(b, c);
    for (int d = 0; d < v->order; ++d) c[d] += t0[d];
    const int64_t pb = T->block_id(c);
    v->nz[b] = T->nz[pb];
    v->blk_off[b] = T->blk_off[pb];
    v->owner[b] = T->owner[pb];
    v->nnz += v->nz[b];
  }
  v->gblk_off = v->blk_off;
  v->packed_elems = T->packed_elems;
  v->storage_elems = T->storage_elems;
  v->parts.assign(v->nblocks, {});
  v->data = T->data;
  v->capacity = T->capacity;
  T->live_views++;
  *out = v;
  return TT_OK;
}



tt_status tt_tensor_set_compact(tt_tensor t, int32_t on) {
  if (!t) return fail(TT_E_ARG, "NULL tensor");
  if (t->view_of) return fail(TT_E_UNSUPPORTED, "a view takes its storage from its parent");
  TT_TRY(check_no_views(t));
  if ((on != 0) != t->compact) {
    t->compact = on != 0;
    apply_storage(t);
    t->version++;
  }
  return TT_OK;
}

tt_status tt_tensor_storage(tt_tensor t, int64_t* storage_elems, const int64_t** storage_off) {
  if (!t) return fail(TT_E_ARG, "NULL tensor");
  if (storage_elems) *storage_elems = t->storage_elems;
  if (storage_off) *storage_off = t->blk_off.data();
  return TT_OK;
}

tt_status tt_tensor_set_owner(tt_tensor t, const int32_t* owner) {
  if (!t || !owner) return fail(TT_E_ARG, "NULL argument");
  if (t->view_of) return fail(TT_E_UNSUPPORTED, "a view takes its owners from its parent");
  TT_TRY(check_no_views(t));
  for (int64_t b = 0; b < t->nblocks; ++b) {
    if (!t->nz[b]) continue;
    if (owner[b] != TT_REPLICATED && (owner[b] < 0 || owner[b] >= t->ctx->nranks))
      return fail(TT_E_ARG, "owner[%lld] = %d out of range", (long long)b, owner[b]);
  }
  for (int64_t b = 0; b < t->nblocks; ++b) t->owner[b] = t->nz[b] ? owner[b] : -1;
  t->parts.assign(t->nblocks, {});
  refresh_parts_view(t);
  apply_storage(t);
  t->version++;
  return TT_OK;
}

tt_status tt_tensor_set_parts(tt_tensor t, int64_t n, const int64_t* blk, const int32_t* lo, const int32_t* hi,
                              const int32_t* owner) {
  if (!t || (n > 0 && (!blk || !lo || !hi || !owner))) return fail(TT_E_ARG, "NULL argument");
  if (t->view_of) return fail(TT_E_UNSUPPORTED, "a view takes its owners from its parent");
  TT_TRY(check_no_views(t));
  std::map<int64_t, std::vector<tt_tensor_s::Part>> np;
  for (int64_t i = 0; i < n; ++i) {
    if (blk[i] < 0 || blk[i] >= t->nblocks || !t->nz[blk[i]])
      return fail(TT_E_ARG, "part %lld: block %lld is not a non-zero block", (long long)i, (long long)blk[i]);
    if (owner[i] < 0 || owner[i] >= t->ctx->nranks) return fail(TT_E_ARG, "part %lld: owner %d out of range", (long long)i, owner[i]);
    np[blk[i]].push_back({lo[i], hi[i], owner[i]});
  }
  for (auto& kv : np) {   // validate: parts tile [0, ext0) in order, non-empty
    int32_t pos = 0;
    for (const auto& p : kv.second) {
      if (p.lo != pos || p.hi <= p.lo) return fail(TT_E_ARG, "parts of block %lld must tile its dim-0 range in order", (long long)kv.first);
      pos = p.hi;
    }
    if (pos != t->ext0(kv.first)) return fail(TT_E_ARG, "parts of block %lld do not cover its dim-0 tile", (long long)kv.first);
  }
  for (auto& kv : np) {
    if (kv.second.size() == 1) {
      t->owner[kv.first] = kv.second[0].owner;
      t->parts[kv.first].clear();
    } else {
      t->owner[kv.first] = TT_SPLIT;
      t->parts[kv.first] = kv.second;
    }
  }
  refresh_parts_view(t);
  apply_storage(t);
  t->version++;
  return TT_OK;
}

tt_status tt_tensor_parts(tt_tensor t, int64_t* n, const int64_t** blk, const int32_t** lo, const int32_t** hi,
                          const int32_t** owner) {
  if (!t || !n) return fail(TT_E_ARG, "NULL argument");
  *n = (int64_t)t->pv_blk.size();
  if (blk) *blk = t->pv_blk.data();
  if (lo) *lo = t->pv_lo.data();
  if (hi) *hi = t->pv_hi.data();
  if (owner) *owner = t->pv_owner.data();
  return TT_OK;
}

tt_status tt_tensor_bind(tt_tensor t, void* ptr, int64_t cap) {
  if (!t) return fail(TT_E_ARG, "NULL tensor");
  if (ptr && ((uintptr_t)ptr % 16) != 0) return fail(TT_E_ARG, "storage must be 16-byte aligned");
  if (ptr && cap < t->storage_elems)
    return fail(TT_E_UNBOUND, "capacity %lld < storage size %lld", (long long)cap, (long long)t->storage_elems);
  t->data = (double*)ptr;
  t->capacity = cap;
  return TT_OK;
}

tt_status tt_tensor_upload(tt_ctx ctx, tt_tensor t, const double* host) {
  NvtxRange nvtx_("tt_tensor_upload");
  TT_TRY(need_device(ctx));
  if (!t || !host) return fail(TT_E_ARG, "NULL argument");
  TT_TRY(check_bound(t, "upload"));
  DeviceGuard dg(ctx->device);
  TT_CUDA(cudaMemcpyAsync(t->data, host, t->storage_elems * 8, cudaMemcpyHostToDevice, ctx->stream));
  return TT_OK;
}

tt_status tt_tensor_download(tt_ctx ctx, tt_tensor t, double* host) {
  NvtxRange nvtx_("tt_tensor_download");
  TT_TRY(need_device(ctx));
  if (!t || !host) return fail(TT_E_ARG, "NULL argument");
  TT_TRY(check_bound(t, "download"));
  DeviceGuard dg(ctx->device);
  TT_CUDA(cudaMemcpyAsync(host, t->data, t->storage_elems * 8, cudaMemcpyDeviceToHost, ctx->stream));
  return TT_OK;
}

tt_status tt_tensor_destroy(tt_tensor t) {
  // device metadata is owned by the context allocation list (freed by tt_ctx_destroy)
  if (t && t->view_of) t->view_of->live_views--;
  if (t && t->sim) {
    std::lock_guard<std::mutex> lk(t->sim->mu);
    auto it = t->sim->reg.find(t->seq);
    if (it != t->sim->reg.end() && it->second[t->sim_rank] == t) {
      it->second[t->sim_rank] = nullptr;
      bool any = false;
      for (tt_tensor u : it->second) any = any || u;
      if (!any) t->sim->reg.erase(it);
    }
  }
  delete t;
  return TT_OK;
}

}  // extern "C"

// =============================================================================================
// element operations (set / add / fill / scalar): segment lists built on the host

namespace {

constexpr int64_t kSegElems = 1 << 15;

struct ElemPlan {
  DevMem mem;                 // workspace regions of the device arrays below
  std::vector<ElemDesc> descs;
  std::vector<Segment> segs;
  std::vector<TileItem> tiles;
  ElemDesc* d_descs = nullptr;
  Segment* d_segs = nullptr;
  TileItem* d_tiles = nullptr;
  double* d_partials = nullptr;
  GatherPlan gp;
  double bytes = 0;
  int64_t blocks = 0;
  int64_t nseg() const { return (int64_t)segs.size(); }
  int64_t ntiles() const { return (int64_t)tiles.size(); }
};

// Fuse adjacent x dims that are adjacent (same order) in y; fill the group extents / y strides of
// one block descriptor.  ext[d] = x block extents, ypos[d] = y dim of x dim d, ystr[e] = y block
// strides by y dim.  Returns the element-op mode of this descriptor.
int fuse_elem(ElemDesc& d, int order, const int32_t* ext, const int* ypos, const int64_t* ystr) {
  int n = 0;
  int64_t gext[TT_MAX_ORDER];
  int last_y[TT_MAX_ORDER];
  for (int q = 0; q < order; ++q) {
    if (n > 0 && ypos[q] == last_y[n - 1] + 1) {
      gext[n - 1] *= ext[q];
      last_y[n - 1] = ypos[q];
    } else {
      gext[n] = ext[q];
      last_y[n] = ypos[q];
      ++n;
    }
  }
  d.n = n;
  d.gy = -1;
  for (int g = 0; g < n; ++g) {
    d.div[g] = make_fastdiv((uint32_t)gext[g]);
    d.y_str[g] = (int32_t)ystr[last_y[g]];
    if (d.y_str[g] == 1) d.gy = g;
  }
  if (n == 1 && d.y_str[0] == 1) d.mode = kElemContig;
  else if (d.y_str[n - 1] == 1 && d.div[n - 1].d >= 8) d.mode = kElemRows;
  else if (d.y_str[n - 1] == 1) d.mode = kElemGeneric;
  else if (d.gy < 0) d.mode = kElemGeneric;
  else d.mode = kElemTranspose;
  return d.mode;
}

// transpose-mode work of a whole block: 32x32 tiles over (gx = innermost X group, gy = the group with
// Y stride 1), one per remaining-group index; bases precomputed (TileItem)
void add_tiles(ElemPlan& ep, const ElemDesc& d) {
  const int gx = d.n - 1, gy = d.gy;
  int64_t xs[TT_MAX_ORDER], acc = 1;
  for (int g = d.n - 1; g >= 0; --g) { xs[g] = acc; acc *= d.div[g].d; }
  int64_t batch = 1;
  for (int g = 0; g < d.n; ++g)
    if (g != gx && g != gy) batch *= d.div[g].d;
  const int ex = (int)d.div[gx].d, ey = (int)d.div[gy].d;
  for (int64_t b = 0; b < batch; ++b) {
    int64_t r = b, xb = 0, yb = 0;
    for (int g = d.n - 1; g >= 0; --g) {
      if (g == gx || g == gy) continue;
      const int64_t c = r % d.div[g].d;
      r /= d.div[g].d;
      xb += c * xs[g];
      yb += c * d.y_str[g];
    }
    for (int ty = 0; ty < ey; ty += 32)
      for (int tx = 0; tx < ex; tx += 32) {
        TileItem t;
        t.x_base = d.x_off + xb + (int64_t)ty * xs[gy] + tx;
        t.y_base = d.y_off < 0 ? -1 : d.y_off + yb + (int64_t)tx * d.y_str[gx] + ty;
        t.nx = std::min(32, ex - tx);
        t.ny = std::min(32, ey - ty);
        t.x_ld = (int32_t)xs[gy];
        t.y_ld = d.y_str[gx];
        ep.tiles.push_back(t);
      }
  }
}

void add_segments(ElemPlan& ep, int32_t desc, int64_t e_begin, int64_t e_end) {
  for (int64_t e = e_begin; e < e_end; e += kSegElems) ep.segs.push_back({desc, 0, e, std::min(e_end, e + kSegElems)});
}

// Appends one block descriptor (mode set by fuse_elem) and its work: 32x32 tiles over the whole block
// for a transpose descriptor (only when the block is processed whole), else segments over `ranges`.
// Modes are per descriptor: blocks of one plan may differ (e.g. a remainder tile of extent 1 makes
// a transposing block generic), and every block's work is kept.
void emit_elem(ElemPlan& ep, ElemDesc& d, bool whole, const std::vector<std::pair<int64_t, int64_t>>& ranges) {
  if (d.mode == kElemTranspose && !whole) d.mode = kElemGeneric;   // tiles need whole blocks
  ep.descs.push_back(d);
  const int32_t di = (int32_t)ep.descs.size() - 1;
  if (d.mode == kElemTranspose) {
    add_tiles(ep, d);
    return;
  }
  for (auto& h : ranges) add_segments(ep, di, h.first, h.second);
}

// whether the dim-0 label of X is also the dim-0 label of Y: then a row range of an X part maps to
// a contiguous row range of the matching Y block
int64_t sub_range_inner(tt_tensor Y, int64_t yb, bool same_dim0, int64_t lo_row, int64_t hi_row, int64_t* e0,
                        int64_t* e1) {
  const int64_t vol = Y->block_volume(yb);
  if (!same_dim0) {
    *e0 = 0;
    *e1 = vol;
    return vol;
  }
  const int64_t inner = vol / Y->ext0(yb);
  *e0 = lo_row * inner;
  *e1 = hi_row * inner;
  return inner;
}

tt_status upload_elem_once(tt_ctx ctx, ElemPlan& ep, bool partials) {
  TT_TRY(dev_alloc(ctx, ep.mem, &ep.d_descs, ep.descs.size()));
  TT_TRY(dev_alloc(ctx, ep.mem, &ep.d_segs, ep.segs.size()));
  if (!ep.descs.empty()) TT_CUDA(cudaMemcpy(ep.d_descs, ep.descs.data(), ep.descs.size() * sizeof(ElemDesc), cudaMemcpyHostToDevice));
  if (!ep.segs.empty()) TT_CUDA(cudaMemcpy(ep.d_segs, ep.segs.data(), ep.segs.size() * sizeof(Segment), cudaMemcpyHostToDevice));
  if (!ep.tiles.empty()) {
    TT_TRY(dev_alloc(ctx, ep.mem, &ep.d_tiles, ep.tiles.size()));
    TT_CUDA(cudaMemcpy(ep.d_tiles, ep.tiles.data(), ep.tiles.size() * sizeof(TileItem), cudaMemcpyHostToDevice));
  }
  if (partials) {
    const int64_t n = ep.nseg() + ep.ntiles();
    TT_TRY(dev_alloc(ctx, ep.mem, &ep.d_partials, (size_t)(n + scalar_scratch_elems(n))));
  }
  return TT_OK;
}

tt_status upload_elem(tt_ctx ctx, ElemPlan& ep, bool partials) {
  tt_status st = upload_elem_once(ctx, ep, partials);
  if (st == TT_E_WORKSPACE && ctx->ws.base) {   // retry from an emptied cache (see ws_make_room)
    ep.mem.release();
    TT_TRY(ws_make_room(ctx));
    st = upload_elem_once(ctx, ep, partials);
  }
  return st;
}

template <class P>
std::shared_ptr<P> cached(tt_ctx ctx, const std::string& key) {
  auto it = ctx->plans.find(key);
  if (it == ctx->plans.end()) return nullptr;
  it->second.tick = ++ctx->plan_tick;
  if (ctx->plan_sink) ctx->plan_sink->push_back(it->second.p);
  return std::static_pointer_cast<P>(it->second.p);
}

void reset_stats(tt_ctx ctx) { ctx->last = tt_stats{}; }

}  // namespace

extern "C" {

tt_status tt_fill_synthetic(tt_ctx ctx, tt_tensor t, uint64_t seed, uint32_t tag, int32_t kind) {
  NvtxRange nvtx_("tt_fill_synthetic");
  TT_TRY(need_ws(ctx));
  if (!t) return fail(TT_E_ARG, "NULL tensor");
  if (kind != TT_KIND_UNIFORM && kind != TT_KIND_INTEGER) return fail(TT_E_ARG, "bad kind %d", kind);
  TT_TRY(check_bound(t, "fill"));
  DeviceGuard dg(ctx->device);
  char keybuf[128];
  snprintf(keybuf, sizeof(keybuf), "fill|%llu.%llu", (unsigned long long)t->uid, (unsigned long long)t->version);
  auto ep = cached<ElemPlan>(ctx, keybuf);
  if (!ep) {
    ep = std::make_shared<ElemPlan>();
    std::vector<int64_t> gstr(t->order);
    int64_t acc = 1;
    for (int d = t->order - 1; d >= 0; --d) { gstr[d] = acc; acc *= t->dims[d]->is->extent; }
    int32_t c[TT_MAX_ORDER];
    std::vector<std::pair<int64_t, int64_t>> hr;
    for (int64_t b = 0; b < t->nblocks; ++b) {
      t->held_ranges(b, ctx->rank, hr);
      if (hr.empty()) continue;
      t->block_coords(b, c);
      ElemDesc d{};
      d.x_off = t->blk_off[b];
      d.y_off = -1;
      d.g_origin = 0;
      d.n = t->order;
      for (int q = 0; q < t->order; ++q) {
        d.div[q] = make_fastdiv((uint32_t)t->dims[q]->size(c[q]));
        d.g_str[q] = gstr[q];
        d.g_origin += t->dims[q]->offsets[c[q]] * gstr[q];
      }
      ep->descs.push_back(d);
      for (auto& r : hr) add_segments(*ep, (int32_t)ep->descs.size() - 1, r.first, r.second);
    }
    TT_TRY(upload_elem(ctx, *ep, false));
    plan_put(ctx, keybuf, ep);
  }
  if (ctx->prepare_only) return TT_OK;
  reset_stats(ctx);
  ElemParams p{};
  p.X = t->data;
  p.descs = ep->d_descs;
  p.segs = ep->d_segs;
  p.order = t->order;
  p.key = seed ^ ((uint64_t)tag * 0x9E3779B97F4A7C15ull);
  p.kind = kind;
  {
    Launch L(ctx, "tt_fill_synthetic");
    TT_CUDA(launch_fill(p, (int64_t)ep->segs.size(), ctx->stream));
  }
  return TT_OK;
}

tt_status tt_set(tt_ctx ctx, tt_tensor C, double alpha) {
  NvtxRange nvtx_("tt_set");
  TT_TRY(need_ws(ctx));
  if (!C) return fail(TT_E_ARG, "NULL tensor");
  TT_TRY(check_bound(C, "C"));
  DeviceGuard dg(ctx->device);
  char keybuf[128];
  snprintf(keybuf, sizeof(keybuf), "set|%llu.%llu", (unsigned long long)C->uid, (unsigned long long)C->version);
  auto ep = cached<ElemPlan>(ctx, keybuf);
  if (!ep) {
    ep = std::make_shared<ElemPlan>();
    std::vector<std::pair<int64_t, int64_t>> hr;
    for (int64_t b = 0; b < C->nblocks; ++b) {
      C->held_ranges(b, ctx->rank, hr);
      if (hr.empty()) continue;
      ElemDesc d{};
      d.x_off = C->blk_off[b];
      d.y_off = -1;
      ep->descs.push_back(d);
      for (auto& r : hr) {
        add_segments(*ep, (int32_t)ep->descs.size() - 1, r.first, r.second);
        ep->bytes += 8.0 * (r.second - r.first);
      }
      ep->blocks++;
    }
    TT_TRY(upload_elem(ctx, *ep, false));
    plan_put(ctx, keybuf, ep);
  }
  if (ctx->prepare_only) return TT_OK;
  reset_stats(ctx);
  ElemParams p{};
  p.X = C->data;
  p.descs = ep->d_descs;
  p.segs = ep->d_segs;
  p.alpha = alpha;
  {
    Launch L(ctx, "tt_set");
    TT_CUDA(launch_set(p, (int64_t)ep->segs.size(), ctx->stream));
  }
  ctx->last.c_blocks = ep->blocks;
  ctx->last.bytes = ep->bytes;
  return TT_OK;
}

tt_status tt_add(tt_ctx ctx, tt_tensor C, const char* cl, double beta, double alpha, tt_tensor A, const char* al) {
  NvtxRange nvtx_("tt_add");
  if (!ctx || !C || !A) return fail(TT_E_ARG, "NULL argument");
  TT_TRY(check_labels(cl, C, "C"));
  TT_TRY(check_labels(al, A, "A"));
  if (C == A) return fail(TT_E_ARG, "C and A must be different tensors");
  std::string c(cl), a(al);
  if (c.size() != a.size()) return fail(TT_E_LABEL, "add needs the same labels on both sides (P173)");
  std::vector<int> perm(c.size());   // C dim d holds the label of A dim perm[d]
  for (size_t d = 0; d < c.size(); ++d) {
    size_t p = a.find(c[d]);
    if (p == std::string::npos) return fail(TT_E_LABEL, "label '%c' of C missing in A (P173)", c[d]);
    if (!same_tiling(C->dims[d], A->dims[p])) return fail(TT_E_TILING, "label '%c' on different tilings (S413)", c[d]);
    perm[d] = (int)p;
  }
  TT_TRY(need_ws(ctx));
  TT_TRY(check_bound(C, "C"));
  TT_TRY(check_bound(A, "A"));
  DeviceGuard dg(ctx->device);
  std::string key = plan_key("add", C, cl, A, al, nullptr, nullptr, beta);
  auto ep = cached<ElemPlan>(ctx, key);
  if (!ep) {
    ep = std::make_shared<ElemPlan>();
    Needs need(ctx->nranks);
    int32_t cc[TT_MAX_ORDER], ac[TT_MAX_ORDER];
    const bool same0 = perm[0] == 0;
    std::vector<std::pair<int64_t, int64_t>> hr, mine;
    for (int64_t b = 0; b < C->nblocks; ++b) {
      if (!C->nz[b]) continue;
      C->block_coords(b, cc);
      for (int d = 0; d < C->order; ++d) ac[perm[d]] = cc[d];
      int64_t ab = A->block_id(ac);
      const int64_t cin = C->block_volume(b) / C->ext0(b);
      for (int r = 0; r < ctx->nranks; ++r) {
        C->held_ranges(b, r, hr);
        if (r == ctx->rank) mine = hr;
        if (!A->nz[ab]) continue;
        for (auto& h : hr) {
          int64_t e0, e1;
          sub_range_inner(A, ab, same0, h.first / cin, h.second / cin, &e0, &e1);
          need[r].push_back({0, ab, e0, e1});
        }
      }
      if (mine.empty()) continue;
      ElemDesc d{};
      d.x_off = C->blk_off[b];
      d.y_off = A->nz[ab] ? A->blk_off[ab] : -1;
      // strides of the A block, by A dim
      int64_t sa[TT_MAX_ORDER], acc = 1;
      for (int q = A->order - 1; q >= 0; --q) { sa[q] = acc; acc *= A->dims[q]->size(ac[q]); }
      int32_t ext[TT_MAX_ORDER];
      for (int q = 0; q < C->order; ++q) ext[q] = (int32_t)C->dims[q]->size(cc[q]);
      fuse_elem(d, C->order, ext, perm.data(), sa);
      const bool whole = mine.size() == 1 && mine[0].first == 0 && mine[0].second == C->block_volume(b);
      emit_elem(*ep, d, whole, mine);
      for (auto& h : mine) ep->bytes += 8.0 * (h.second - h.first) * ((beta != 0.0) + 1 + (A->nz[ab] ? 1 : 0));
      ep->blocks++;
    }
    TT_TRY(build_gather(ctx, need, {A}, ep->gp));
    TT_TRY(upload_elem(ctx, *ep, false));
    plan_put(ctx, key, ep);
  }
  if (ctx->prepare_only) return TT_OK;
  reset_stats(ctx);
  TT_TRY(run_gather(ctx, ep->gp, {A}));
  ElemParams p{};
  p.X = C->data;
  p.Y = A->data;
  p.descs = ep->d_descs;
  p.segs = ep->d_segs;
  p.tiles = ep->d_tiles;
  p.order = C->order;
  p.alpha = alpha;
  p.beta = beta;
  {
    Launch L(ctx, "tt_add");
    TT_CUDA(launch_add(p, ep->nseg(), ep->ntiles(), ctx->stream));
  }
  ctx->last.c_blocks = ep->blocks;
  ctx->last.bytes = ep->bytes;
  ctx->last.gathered_bytes = ep->gp.recv_bytes;
  return TT_OK;
}

tt_status tt_contract_scalar(tt_ctx ctx, double alpha, tt_tensor A, const char* al, tt_tensor B, const char* bl,
                             double* result) {
  NvtxRange nvtx_("tt_contract_scalar");
  if (!ctx || !A || !B || !result) return fail(TT_E_ARG, "NULL argument");
  TT_TRY(check_labels(al, A, "A"));
  TT_TRY(check_labels(bl, B, "B"));
  std::string a(al), b(bl);
  if (a.size() != b.size()) return fail(TT_E_LABEL, "scalar contraction needs the same label set in A and B");
  std::vector<int> perm(a.size());   // A dim d holds the label of B dim perm[d]
  for (size_t d = 0; d < a.size(); ++d) {
    size_t p = b.find(a[d]);
    if (p == std::string::npos) return fail(TT_E_LABEL, "label '%c' of A missing in B", a[d]);
    if (!same_tiling(A->dims[d], B->dims[p])) return fail(TT_E_TILING, "label '%c' on different tilings (S413)", a[d]);
    perm[d] = (int)p;
  }
  TT_TRY(need_ws(ctx));
  TT_TRY(check_bound(A, "A"));
  TT_TRY(check_bound(B, "B"));
  DeviceGuard dg(ctx->device);
  std::string key = plan_key("scalar", A, al, B, bl, nullptr, nullptr, 0.0);
  auto ep = cached<ElemPlan>(ctx, key);
  if (!ep) {
    ep = std::make_shared<ElemPlan>();
    Needs need(ctx->nranks);
    int32_t ac[TT_MAX_ORDER], bc[TT_MAX_ORDER];
    const bool same0 = perm[0] == 0;
    for (int64_t blk = 0; blk < A->nblocks; ++blk) {
      if (!A->nz[blk]) continue;
      A->block_coords(blk, ac);
      for (int d = 0; d < A->order; ++d) bc[perm[d]] = ac[d];
      int64_t bb = B->block_id(bc);
      if (!B->nz[bb]) continue;
      // the rank that sums a piece of this pair: A's owner of the piece (replicated A blocks: rank 0)
      std::vector<std::pair<int32_t, std::pair<int64_t, int64_t>>> who;
      if (A->parts[blk].empty()) {
        who.push_back({A->owner[blk] == TT_REPLICATED ? 0 : A->owner[blk], {0, A->block_volume(blk)}});
      } else {
        const int64_t inner = A->block_volume(blk) / A->ext0(blk);
        for (const auto& pt : A->parts[blk]) who.push_back({pt.owner, {pt.lo * inner, pt.hi * inner}});
      }
      const int64_t ain = A->block_volume(blk) / A->ext0(blk);
      std::vector<std::pair<int64_t, int64_t>> mine;
      for (auto& w : who) {
        int64_t e0, e1;
        sub_range_inner(B, bb, same0, w.second.first / ain, w.second.second / ain, &e0, &e1);
        need[w.first].push_back({1, bb, e0, e1});
        if (w.first == ctx->rank) mine.push_back(w.second);
      }
      if (mine.empty()) continue;
      ElemDesc d{};
      d.x_off = A->blk_off[blk];
      d.y_off = B->blk_off[bb];
      int64_t sb[TT_MAX_ORDER], acc = 1;
      for (int q = B->order - 1; q >= 0; --q) { sb[q] = acc; acc *= B->dims[q]->size(bc[q]); }
      int32_t ext[TT_MAX_ORDER];
      for (int q = 0; q < A->order; ++q) ext[q] = (int32_t)A->dims[q]->size(ac[q]);
      fuse_elem(d, A->order, ext, perm.data(), sb);
      const bool whole = mine.size() == 1 && mine[0].first == 0 && mine[0].second == A->block_volume(blk);
      emit_elem(*ep, d, whole, mine);
      for (auto& h : mine) ep->bytes += 16.0 * (h.second - h.first);
      ep->blocks++;
    }
    TT_TRY(build_gather(ctx, need, {A, B}, ep->gp));
    TT_TRY(upload_elem(ctx, *ep, true));
    plan_put(ctx, key, ep);
  }
  if (ctx->prepare_only) return TT_OK;
  reset_stats(ctx);
  TT_TRY(run_gather(ctx, ep->gp, {A, B}));
  ElemParams p{};
  p.X = A->data;
  p.Y = B->data;
  p.descs = ep->d_descs;
  p.segs = ep->d_segs;
  p.order = A->order;
  p.tiles = ep->d_tiles;
  p.partials = ep->d_partials;
  double* dst = ctx->scalar_dev_out ? ctx->scalar_dev_out : ctx->d_scalar;
  const int64_t npart = ep->nseg() + ep->ntiles();
  {
    Launch L(ctx, "tt_scalar_partials");
    TT_CUDA(launch_scalar_partials(p, ep->nseg(), ep->ntiles(), ctx->stream));
  }
  {
    Launch L(ctx, "tt_scalar_final");
    TT_CUDA(launch_scalar_final(ep->d_partials, npart, alpha, dst, ep->d_partials + npart, ctx->stream));
  }
  TT_TRY(allreduce_sum(ctx, dst, ctx->stream));
  if (!ctx->scalar_dev_out) {   // inside a captured graph the scheduler copies the device slot later
    TT_CUDA(cudaMemcpyAsync(result, dst, 8, cudaMemcpyDeviceToHost, ctx->stream));
    TT_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  ctx->last.c_blocks = ep->blocks;
  ctx->last.bytes = ep->bytes;
  ctx->last.flops = ep->bytes / 8.0;   // one multiply-add per element pair
  ctx->last.gathered_bytes = ep->gp.recv_bytes;
  return TT_OK;
}

}  // extern "C"

// =============================================================================================
// contraction

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  return fn;
}

// 2-D tensor map of a packed buffer viewed as [rows][cols] doubles
tt_status encode_2d(CUtensorMap* m, const double* base, int64_t cols, int64_t rows, uint32_t box_cols, uint32_t box_rows,
                    bool swizzle128) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(TT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 8};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TT_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TT_OK;
}

// 3-D tensor map of a dense row-major array; dims innermost first (doubles), box likewise, no swizzle
tt_status encode_3d(CUtensorMap* m, const double* base, const int64_t* dims3, const uint32_t* box3) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(TT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)dims3[0], (cuuint64_t)dims3[1], (cuuint64_t)dims3[2]};
  cuuint64_t strides[2] = {(cuuint64_t)dims3[0] * 8, (cuuint64_t)(dims3[0] * dims3[1]) * 8};
  cuuint32_t box[3] = {box3[0], box3[1], box3[2]}, es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TT_E_CUDA, "cuTensorMapEncodeTiled (3-D) failed (%d)", (int)r);
  return TT_OK;
}

// 4-D tensor map of a dense row-major array; dims innermost first (doubles), box likewise
tt_status encode_4d(CUtensorMap* m, const double* base, const int64_t* dims4, const uint32_t* box4) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(TT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], es[4] = {1, 1, 1, 1};
  cuuint64_t acc = 8;
  for (int q = 0; q < 4; ++q) {
    dims[q] = (cuuint64_t)dims4[q];
    box[q] = box4[q];
    if (q > 0) strides[q - 1] = acc;
    acc *= (cuuint64_t)dims4[q];
  }
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TT_E_CUDA, "cuTensorMapEncodeTiled (4-D) failed (%d)", (int)r);
  return TT_OK;
}

// uniform extent of a fused label group over every non-zero block of T (-1 if it varies)
int64_t uniform_group_extent(tt_tensor T, const std::vector<int>& tdims) {
  int64_t e = -1;
  int32_t c[TT_MAX_ORDER];
  for (int64_t b = 0; b < T->nblocks; ++b) {
    if (!T->nz[b]) continue;
    T->block_coords(b, c);
    int64_t x = 1;
    for (int d : tdims) x *= T->dims[d]->size(c[d]);
    if (e < 0) e = x;
    else if (e != x) return -1;
  }
  return e;
}

tt_status build_contract_plan(tt_ctx ctx, tt_tensor C, tt_tensor A, tt_tensor B, double beta, ContractPlan& pl,
                              const ContractOpts& opts = ContractOpts()) {
  const Analysis& an = pl.an;
  enumerate_tasks(an, C, A, B, pl.ht);
  const HostTasks& ht = pl.ht;
  std::vector<tt_tis> lt(an.uni.size());
  for (size_t u = 0; u < an.uni.size(); ++u) lt[u] = label_tis(an, (int)u, C, A);
  // C parts computed per rank (owner-computes); input ranges read per rank.  When C is row-split
  // and C's dim-0 label is also the dim-0 label of A (B), only the matching rows of A (B) are read.
  Needs need(ctx->nranks);
  const bool a_same0 = an.a_lab[0] == 0, b_same0 = an.b_lab[0] == 0;
  const int bop = (A == B) ? 0 : 1;   // A and B may be the same tensor (same storage)
  std::vector<std::pair<int64_t, int64_t>> hr;
  if (opts.local) {
    std::map<int64_t, int> g_of;
    for (size_t g = 0; g < ht.cblk.size(); ++g) g_of[ht.cblk[g]] = (int)g;
    for (const PartSel& ps : opts.sel) {
      auto it = g_of.find(ps.blk);
      if (it == g_of.end()) return fail(TT_E_ARG, "selected C block %lld is not a non-zero block", (long long)ps.blk);
      pl.my.push_back({it->second, ps.lo, ps.hi});
    }
  } else {
    for (size_t g = 0; g < ht.cblk.size(); ++g) {
      const int64_t cb = ht.cblk[g];
      const int64_t cin = C->block_volume(cb) / C->ext0(cb);
      for (int r = 0; r < ctx->nranks; ++r) {
        C->held_ranges(cb, r, hr);
        for (auto& h : hr) {
          const int64_t lo = h.first / cin, hi = h.second / cin;
          if (r == ctx->rank) pl.my.push_back({(int)g, lo, hi});
          if (opts.no_gather) continue;
          for (int64_t t = ht.ptr[g]; t < ht.ptr[g + 1]; ++t) {
            int64_t e0, e1;
            sub_range_inner(A, ht.a_blk[t], a_same0, lo, hi, &e0, &e1);
            need[r].push_back({0, ht.a_blk[t], e0, e1});
            sub_range_inner(B, ht.b_blk[t], b_same0, lo, hi, &e0, &e1);
            need[r].push_back({bop, ht.b_blk[t], e0, e1});
          }
        }
      }
    }
    if (!opts.no_gather) {
      if (A == B) TT_TRY(build_gather(ctx, need, {A}, pl.gp));
      else TT_TRY(build_gather(ctx, need, {A, B}, pl.gp));
    }
  }
  // stats for this rank
  {
    std::vector<char> ua(A->nblocks, 0), ub(B->nblocks, 0);
    for (const auto& mp : pl.my) {
      const int g = mp.g;
      const double frac = (double)(mp.hi - mp.lo) / (double)C->ext0(ht.cblk[g]);
      pl.flops += (double)ht.cost[g] * frac;
      pl.tasks += ht.ptr[g + 1] - ht.ptr[g];
      pl.bytes += 8.0 * C->block_volume(ht.cblk[g]) * frac * (1 + (beta != 0.0));
      for (int64_t t = ht.ptr[g]; t < ht.ptr[g + 1]; ++t) {
        if (!ua[ht.a_blk[t]]) { ua[ht.a_blk[t]] = 1; pl.bytes += 8.0 * A->block_volume(ht.a_blk[t]) * (a_same0 ? frac : 1.0); }
        if (!ub[ht.b_blk[t]]) { ub[ht.b_blk[t]] = 1; pl.bytes += 8.0 * B->block_volume(ht.b_blk[t]) * (b_same0 ? frac : 1.0); }
      }
    }
  }
  if (ctx->device < 0) return TT_OK;

  // ---- device task-list builder (count -> scan -> fill)
  TT_TRY(ensure_dev(C));
  TT_TRY(ensure_dev(A));
  TT_TRY(ensure_dev(B));
  const int64_t ncb = (int64_t)ht.cblk.size(), ntasks = (int64_t)ht.a_blk.size();
  int64_t *d_cblocks, *d_counts;
  DevMem tmp;   // builder scratch, retired when the plan is built
  TT_TRY(dev_alloc(ctx, tmp, &d_cblocks, ncb));
  TT_TRY(dev_alloc(ctx, tmp, &d_counts, ncb));
  TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_ptr, ncb + 1));
  TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_ablk, ntasks));
  TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_bblk, ntasks));
  TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_tasks, ntasks));
  TT_CUDA(cudaMemcpy(d_cblocks, ht.cblk.data(), ncb * 8, cudaMemcpyHostToDevice));
  BuildParams bp{};
  bp.nc = an.nc;
  bp.nk = an.nk;
  for (int d = 0; d < an.nc; ++d) bp.c_grid[d] = C->grid[d];
  bp.ntuples = 1;
  for (int l = 0; l < an.nk; ++l) { bp.k_grid[l] = lt[an.nc + l]->ntiles(); bp.ntuples *= bp.k_grid[l]; }
  bp.a_order = A->order;
  bp.b_order = B->order;
  for (int d = 0; d < A->order; ++d) { bp.a_lab[d] = an.a_lab[d]; bp.a_grid[d] = A->grid[d]; }
  for (int d = 0; d < B->order; ++d) { bp.b_lab[d] = an.b_lab[d]; bp.b_grid[d] = B->grid[d]; }
  for (size_t u = 0; u < an.uni.size(); ++u) {
    bp.a_pos[u] = an.a_pos[u];
    bp.b_pos[u] = an.b_pos[u];
    bp.lab_toff[u] = (int)u < an.nc ? C->d_toff[u] : A->d_toff[an.a_pos[u]];
  }
  bp.a_nz = A->d_nz;
  bp.b_nz = B->d_nz;
  bp.a_boff = A->d_blk_off;
  bp.b_boff = B->d_blk_off;
  int nl = 0;
  auto put = [&](const std::vector<std::vector<int>>& G, int32_t* first, int32_t* cnt) {
    for (size_t g = 0; g < G.size(); ++g) {
      first[g] = nl;
      cnt[g] = (int32_t)G[g].size();
      for (int u : G[g]) bp.glab[nl++] = u;
    }
    return (int32_t)G.size();
  };
  bp.nM = put(an.mg, bp.m_first, bp.m_cnt);
  bp.nN = put(an.ng, bp.n_first, bp.n_cnt);
  bp.nK = put(an.kg, bp.k_first, bp.k_cnt);
  bp.cblocks = d_cblocks;
  bp.ncb = (int32_t)ncb;
  bp.counts = d_counts;
  bp.ptr = pl.d_ptr;
  bp.a_blk = pl.d_ablk;
  bp.b_blk = pl.d_bblk;
  bp.tasks = pl.d_tasks;
  {
    Launch L(ctx, "tt_build_count");
    TT_CUDA(launch_build_count(bp, ctx->stream));
  }
  {
    Launch L(ctx, "tt_build_scan");
    TT_CUDA(launch_build_scan(bp, ctx->stream));
  }
  {
    Launch L(ctx, "tt_build_fill");
    TT_CUDA(launch_build_fill(bp, ctx->stream));
  }
  int64_t dev_total = -1;
  TT_CUDA(cudaMemcpyAsync(&dev_total, pl.d_ptr + ncb, 8, cudaMemcpyDeviceToHost, ctx->stream));
  TT_CUDA(cudaStreamSynchronize(ctx->stream));
  if (dev_total != ntasks)
    return fail(TT_E_STATE, "device task builder produced %lld tasks, host enumerator %lld", (long long)dev_total,
                (long long)ntasks);
  pl.device_built = true;

  // ---- tile variant: greedy list-scheduling estimate of the makespan
  // GEMM row / column ranges of every part (the split dim 0 of C is the outermost label of the first
  // M group when it comes from A, else of the first N group)
  const bool split_in_m = an.a_pos[0] >= 0;
  std::vector<int64_t> Mb(pl.my.size()), Me(pl.my.size()), Nb(pl.my.size()), Ne(pl.my.size());
  int32_t cc[TT_MAX_ORDER];
  for (size_t i = 0; i < pl.my.size(); ++i) {
    const auto& mp = pl.my[i];
    C->block_coords(ht.cblk[mp.g], cc);
    int64_t M = 1, N = 1;
    for (int u = 0; u < an.nc; ++u) (an.a_pos[u] >= 0 ? M : N) *= lt[u]->size(cc[u]);
    const int64_t e0 = lt[0]->size(cc[0]);
    Mb[i] = 0; Me[i] = M; Nb[i] = 0; Ne[i] = N;
    if (split_in_m) { Mb[i] = mp.lo * (M / e0); Me[i] = mp.hi * (M / e0); }
    else { Nb[i] = mp.lo * (N / e0); Ne[i] = mp.hi * (N / e0); }
  }
  // 16-B copies: the operand's innermost dim is the innermost label of its contiguous group, with
  // even extent in every tile
  {
    auto even = [&](int u) {
      for (int t = 0; t < lt[u]->ntiles(); ++t)
        if (lt[u]->size(t) % 2) return false;
      return true;
    };
    const int a_last = an.a_lab.back(), b_last = an.b_lab.back();
    const int a_grp_last = an.a_kc ? an.kg.back().back() : an.mg.back().back();
    const int b_grp_last = an.b_nc ? an.ng.back().back() : an.kg.back().back();
    pl.a_vec = a_last == a_grp_last && even(a_last);
    pl.b_vec = b_last == b_grp_last && even(b_last);
  }
  // TMA producer (warp-specialised family): every A block is one row-major [M][K] matrix -- A's labels
  // are the M groups' labels (C order) followed by the K groups' labels -- with the same K extent in
  // every block (a multiple of 16: no K tail), and every B block is [K][N] (K labels then N labels,
  // same even N extent) or [N][K] (N labels then K labels: the implicit operand's X(q,s,L)).  Then the
  // packed buffers are [rows][K] / [rows][N|K] matrices and the GEMM row / column index is the row of
  // the block's matrix.  C's label order is free: several M or N groups use the multi-group epilogue.
  {
    const char* ft = getenv("TT_TMA");
    const bool allow = !ft || atoi(ft) != 0;
    std::vector<int> mlab, nlab, klab;
    for (auto& gr : an.mg) mlab.insert(mlab.end(), gr.begin(), gr.end());
    for (auto& gr : an.ng) nlab.insert(nlab.end(), gr.begin(), gr.end());
    for (auto& gr : an.kg) klab.insert(klab.end(), gr.begin(), gr.end());
    auto cat = [](const std::vector<int>& x, const std::vector<int>& y) {
      std::vector<int> r(x);
      r.insert(r.end(), y.begin(), y.end());
      return r;
    };
    const bool a_mk = an.a_lab == cat(mlab, klab);
    const bool b_kn = an.b_lab == cat(klab, nlab), b_nk = an.b_lab == cat(nlab, klab);
    if (allow && !A->view_of && !B->view_of && a_mk && (b_kn || b_nk) && !ht.K.empty() && !klab.empty() &&
        !mlab.empty() && !nlab.empty()) {
      std::vector<int> ak, bn;
      for (int u : klab) ak.push_back(an.a_pos[u]);
      for (int u : nlab) bn.push_back(an.b_pos[u]);
      const int64_t K = uniform_group_extent(A, ak), N = uniform_group_extent(B, bn);
      // even rows (16-byte TMA strides); K tails are TMA out-of-bounds zero fill in both views
      bool ok = K > 0 && N > 0 && K % 2 == 0 && (b_nk || N % 2 == 0);
      for (int32_t k : ht.K) ok = ok && k == K;
      // every stored block starts on a row of its matrix view (no alignment pads between blocks)
      for (int64_t b = 0; ok && b < A->nblocks; ++b)
        if (A->nz[b] && A->blk_off[b] >= 0) ok = A->blk_off[b] % K == 0;
      const int64_t bunit = b_nk ? K : K * N;
      for (int64_t b = 0; ok && b < B->nblocks; ++b)
        if (B->nz[b] && B->blk_off[b] >= 0) ok = B->blk_off[b] % bunit == 0;
      if (ok) {
        pl.tma = true;
        pl.tma_k = K;
        pl.tma_n = b_nk ? K : N;
        pl.tma_mode = (b_nk ? 1 : 0) | ((an.mg.size() > 1 || an.ng.size() > 1) ? 2 : 0);
      }
    }
  }
  // ---- split-K: when the whole contraction (all ranks) has too few output elements to give every
  // SM two tiles, each C block's task list is cut into up to S contiguous chunks of balanced K that
  // run as separate work items writing partial sums, reduced in chunk order afterwards.  The cut
  // depends only on the block's own task list and the global output size -- not on the rank count,
  // the row split or the kernel variant -- so results stay independent of them (R12).
  std::vector<std::vector<int64_t>> chunks(ht.cblk.size());   // task boundaries per C block
  {
    double e_total = 0;
    for (size_t g = 0; g < ht.cblk.size(); ++g)
      if (ht.ptr[g + 1] > ht.ptr[g]) e_total += (double)C->block_volume(ht.cblk[g]);
    const double target = (double)ctx->sm_count * 2.0 * 80.0 * 80.0;
    int64_t s_target = 1;
    if (e_total > 0 && e_total < target) s_target = std::min<int64_t>(64, (int64_t)std::ceil(target / e_total));
    const char* fs = getenv("TT_SPLITK");   // testing / tuning override of the chunk count
    const bool forced = fs != nullptr;
    if (forced) s_target = std::max(1, atoi(fs));
    for (const auto& mp : pl.my) {
      const int g = mp.g;
      auto& cb = chunks[g];
      if (!cb.empty()) continue;
      int64_t ktot = 0;
      for (int64_t t = ht.ptr[g]; t < ht.ptr[g + 1]; ++t) ktot += ht.K[t];
      const int64_t ntk = ht.ptr[g + 1] - ht.ptr[g];
      const int64_t S = std::max<int64_t>(1, std::min<int64_t>({s_target, ntk, forced ? ntk : ktot / 512}));
      cb.push_back(ht.ptr[g]);
      int64_t cum = 0, j = 1;
      for (int64_t t = ht.ptr[g]; t < ht.ptr[g + 1] && j < S; ++t) {
        cum += ht.K[t];
        if (cum * S >= j * ktot && t + 1 < ht.ptr[g + 1]) {   // boundary after task t
          cb.push_back(t + 1);
          while (j < S && cum * S >= j * ktot) ++j;
        }
      }
      cb.push_back(ht.ptr[g + 1]);
    }
  }
  double best = -1;
  std::vector<double> model_mk;
  for (int v = 0; v < n_variants(); ++v) {
    VariantInfo vi = variant_info(v);
    std::vector<double> items;
    for (size_t i = 0; i < pl.my.size(); ++i) {
      const auto& cb = chunks[pl.my[i].g];
      const int64_t nit = ((Me[i] - Mb[i] + vi.bm - 1) / vi.bm) * ((Ne[i] - Nb[i] + vi.bn - 1) / vi.bn);
      for (size_t h = 0; h + 1 < cb.size(); ++h) {
        double kst = 0;
        for (int64_t t = cb[h]; t < cb[h + 1]; ++t) kst += (double)((ht.K[t] + vi.bk - 1) / vi.bk);
        const double c = (double)vi.bm * vi.bn * vi.bk * std::max(kst, 1.0) * vi.ctas_per_sm /
                         variant_efficiency(v, pl.tma && v >= num_contract_variants());
        for (int64_t i = 0; i < nit; ++i) items.push_back(c);
      }
    }
    std::sort(items.begin(), items.end(), std::greater<double>());
    std::priority_queue<double, std::vector<double>, std::greater<double>> slots;
    for (int s = 0; s < ctx->sm_count * vi.ctas_per_sm; ++s) slots.push(0.0);
    double mk = 0;
    for (double c : items) {
      double t0 = slots.top();
      slots.pop();
      slots.push(t0 + c);
      mk = std::max(mk, t0 + c);
    }
    model_mk.push_back(mk);
    if (best < 0 || mk < best * 0.99) {  // prefer earlier variants unless >1% better
      best = mk;
      pl.variant = v;
    }
  }
  // runner-up among the warp-specialised variants (candidate for measured autotuning in tt_contract)
  pl.alt_variant = -1;
  for (int v = num_contract_variants(); v < n_variants(); ++v)
    if (v != pl.variant && (pl.alt_variant < 0 || model_mk[v] < model_mk[pl.alt_variant])) pl.alt_variant = v;
  if (const char* fv = getenv("TT_FORCE_VARIANT")) pl.variant = atoi(fv) % n_variants();
  if (opts.force_variant >= 0) pl.variant = opts.force_variant;
  if (pl.variant < num_contract_variants()) pl.tma = false;   // the classic family has no TMA path
  VariantInfo vi = variant_info(pl.variant);

  // ---- groups + work items (groups by cost desc, block id asc)
  std::vector<size_t> order(pl.my.size());
  std::iota(order.begin(), order.end(), 0);
  auto pcost = [&](size_t i) {
    const auto& mp = pl.my[i];
    return (double)ht.cost[mp.g] * (double)(mp.hi - mp.lo) / (double)C->ext0(ht.cblk[mp.g]);
  };
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
    if (pcost(x) != pcost(y)) return pcost(x) > pcost(y);
    return ht.cblk[pl.my[x].g] < ht.cblk[pl.my[y].g];
  });
  std::vector<CGroupDesc> groups;
  std::vector<WorkItem> work;
  for (size_t oi : order) {
    const int g = pl.my[oi].g;
    CGroupDesc gd{};
    int64_t cb = ht.cblk[g];
    C->block_coords(cb, cc);
    gd.c_off = C->blk_off[cb];
    gd.M = (int32_t)Me[oi];
    gd.N = (int32_t)Ne[oi];
    gd.m_begin = (int32_t)Mb[oi];
    gd.n_begin = (int32_t)Nb[oi];
    gd.task_begin = (int32_t)ht.ptr[g];
    gd.task_end = (int32_t)ht.ptr[g + 1];
    int64_t sc[TT_MAX_ORDER], acc = 1;
    for (int d = an.nc - 1; d >= 0; --d) { sc[d] = acc; acc *= lt[d]->size(cc[d]); }
    for (int i = 0; i < kMaxGroup; ++i) { gd.mext[i] = gd.next[i] = 1; gd.cm_str[i] = gd.cn_str[i] = 0; }
    for (size_t i = 0; i < an.mg.size(); ++i) {
      int32_t e = 1;
      for (int u : an.mg[i]) e *= (int32_t)lt[u]->size(cc[u]);
      gd.mext[i] = e;
      gd.cm_str[i] = (int32_t)sc[an.mg[i].back()];
    }
    for (size_t i = 0; i < an.ng.size(); ++i) {
      int32_t e = 1;
      for (int u : an.ng[i]) e *= (int32_t)lt[u]->size(cc[u]);
      gd.next[i] = e;
      gd.cn_str[i] = (int32_t)sc[an.ng[i].back()];
    }
    const auto& ch = chunks[g];
    const int64_t nch = (int64_t)ch.size() - 1;
    const int32_t mtn = (gd.M - gd.m_begin + vi.bm - 1) / vi.bm, ntn = (gd.N - gd.n_begin + vi.bn - 1) / vi.bn;
    if (nch > 1) {
      const int64_t bvol = (C->block_volume(ht.cblk[g]) + 1) / 2 * 2;
      pl.splits.push_back({gd.c_off, pl.partial_elems, bvol, (int32_t)groups.size(), (int32_t)nch});
    }
    for (int64_t h = 0; h < nch; ++h) {
      CGroupDesc gc = gd;
      gc.task_begin = (int32_t)ch[h];
      gc.task_end = (int32_t)ch[h + 1];
      int64_t st = 0;
      for (int64_t t = ch[h]; t < ch[h + 1]; ++t) st += (ht.K[t] + vi.bk - 1) / vi.bk;
      gc.nstages = (int32_t)st;
      if (nch > 1) {
        gc.flags = kGroupPartial;
        gc.c_off = pl.partial_elems + h * pl.splits.back().vol;
      }
      const int32_t gi = (int32_t)groups.size();
      groups.push_back(gc);
      for (int32_t mt = 0; mt < mtn; ++mt)
        for (int32_t nt = 0; nt < ntn; ++nt) work.push_back({gi, mt, nt});
    }
    if (nch > 1) pl.partial_elems += nch * pl.splits.back().vol;
  }
  pl.nwork = (int64_t)work.size();
  {
    // persistent CTAs pay off when items are short (pipeline fill and epilogue are a visible share);
    // long items keep the hardware's dynamic block scheduling (better for uneven item costs)
    double st_sum = 0;
    for (const WorkItem& w : work) st_sum += groups[w.group].nstages;
    pl.persistent = !work.empty() && st_sum / (double)work.size() < 512.0;
    if (const char* fp = getenv("TT_PERSISTENT")) pl.persistent = atoi(fp) != 0;
  }
  TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_groups, groups.size()));
  TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_work, work.size()));
  if (!groups.empty()) TT_CUDA(cudaMemcpy(pl.d_groups, groups.data(), groups.size() * sizeof(CGroupDesc), cudaMemcpyHostToDevice));
  if (!work.empty()) TT_CUDA(cudaMemcpy(pl.d_work, work.data(), work.size() * sizeof(WorkItem), cudaMemcpyHostToDevice));
  if (!pl.splits.empty()) {
    TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_splits, pl.splits.size()));
    TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_partials, (size_t)pl.partial_elems));
    TT_CUDA(cudaMemcpy(pl.d_splits, pl.splits.data(), pl.splits.size() * sizeof(SplitDesc), cudaMemcpyHostToDevice));
  }
  return TT_OK;
}

tt_status get_contract_plan(tt_ctx ctx, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                            const char* bl, double beta, std::shared_ptr<ContractPlan>& out, bool* cached_flag,
                            const ContractOpts& opts = ContractOpts()) {
  Analysis an;
  TT_TRY(analyse(C, cl, A, al, B, bl, an));
  if (C == A || C == B) return fail(TT_E_ARG, "C must not alias A or B");
  std::string key = plan_key("contract", C, cl, A, al, B, bl, beta) + opts.tag;
  out = cached<ContractPlan>(ctx, key);
  if (cached_flag) *cached_flag = out != nullptr;
  if (out) return TT_OK;
  auto pl = std::make_shared<ContractPlan>();
  pl->an = an;
  DeviceGuard dg(ctx->device);
  tt_status st = build_contract_plan(ctx, C, A, B, beta, *pl, opts);
  if (st == TT_E_WORKSPACE && ctx->ws.base) {   // the plan's own earlier arrays may split the free space
    pl.reset();
    TT_TRY(ws_make_room(ctx));
    pl = std::make_shared<ContractPlan>();
    pl->an = an;
    st = build_contract_plan(ctx, C, A, B, beta, *pl, opts);
  }
  TT_TRY(st);
  plan_put(ctx, key, pl);
  out = pl;
  return TT_OK;
}

// the DMMA contraction kernel of a plan (no gather)
tt_status launch_plan(tt_ctx ctx, const ContractPlan& pl, tt_tensor C, const char* cl, double beta, double alpha,
                      tt_tensor A, const char* al, tt_tensor B, const char* bl) {
  ContractParams p{};
  p.A = A->data;
  p.B = B->data;
  p.C = C->data;
  p.P = pl.d_partials;
  p.groups = pl.d_groups;
  p.tasks = pl.d_tasks;
  p.work = pl.d_work;
  p.nM = (int32_t)pl.an.mg.size();
  p.nN = (int32_t)pl.an.ng.size();
  p.nK = (int32_t)pl.an.kg.size();
  p.alpha = alpha;
  p.beta = beta;
  p.nwork = pl.nwork;
  p.sm_count = ctx->sm_count;
  p.persistent = pl.persistent ? 1 : 0;
  p.tma_n = (int32_t)pl.tma_n;
  const std::string nm = std::string("tt_contract_dmma[") + cl + "=" + al + "*" + bl + "]";
  {
    Launch L(ctx, nm.c_str());
    if (pl.tma) {
      // (re-)encode the tensor maps when the bound storage changed
      ContractPlan& mp = const_cast<ContractPlan&>(pl);
      if (mp.map_ptr[0] != A->data || mp.map_ptr[1] != B->data) {
        const VariantInfo vi = variant_info(pl.variant);
        TT_TRY(encode_2d(&mp.maps[0], A->data, pl.tma_k, A->storage_elems / pl.tma_k, 16, (uint32_t)vi.bm, true));
        if (pl.tma_mode & 1) {   // [N][K] B: {16 k, BN rows} boxes, swizzled like A
          TT_TRY(encode_2d(&mp.maps[1], B->data, pl.tma_n, B->storage_elems / pl.tma_n, 16, (uint32_t)vi.bn, true));
        } else {                 // [K][N] B: [blocks][K][N], boxes {BN+2 n, 16 k, 1 block}
          const int64_t d3[3] = {pl.tma_n, pl.tma_k, B->storage_elems / (pl.tma_n * pl.tma_k)};
          const uint32_t b3[3] = {(uint32_t)vi.bn + 2, 16, 1};
          TT_TRY(encode_3d(&mp.maps[1], B->data, d3, b3));
        }
        mp.map_ptr[0] = A->data;
        mp.map_ptr[1] = B->data;
      }
      TT_CUDA(launch_contract_tma(pl.variant - num_contract_variants(), pl.tma_mode, p, pl.maps, pl.nwork, ctx->stream));
    } else if (pl.variant < num_contract_variants())
      TT_CUDA(launch_contract(pl.variant, pl.an.a_kc, pl.an.b_nc, p, pl.nwork, ctx->stream));
    else
      TT_CUDA(launch_contract_ws(pl.variant - num_contract_variants(), pl.an.a_kc, pl.an.b_nc, pl.a_vec, pl.b_vec, p,
                                 pl.nwork, ctx->stream));
  }
  if (!pl.splits.empty()) {
    const std::string rn = std::string("tt_contract_reduce[") + cl + "=" + al + "*" + bl + "]";
    Launch R(ctx, rn.c_str());
    TT_CUDA(launch_split_reduce(pl.d_partials, C->data, pl.d_groups, pl.d_splits, (int32_t)pl.splits.size(),
                                p.nM, p.nN, alpha, beta, ctx->stream));
  }
  return TT_OK;
}

}  // namespace

extern "C" {

tt_status tt_contract(tt_ctx ctx, tt_tensor C, const char* cl, double beta, double alpha, tt_tensor A,
                      const char* al, tt_tensor B, const char* bl) {
  NvtxRange nvtx_("tt_contract");
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  std::shared_ptr<ContractPlan> pl;
  bool was_cached = false;
  TT_TRY(get_contract_plan(ctx, C, cl, A, al, B, bl, beta, pl, &was_cached));
  TT_TRY(need_ws(ctx));
  if (ctx->prepare_only) return TT_OK;
  TT_TRY(check_bound(C, "C"));
  TT_TRY(check_bound(A, "A"));
  TT_TRY(check_bound(B, "B"));
  DeviceGuard dg(ctx->device);
  reset_stats(ctx);
  if (pl->prefetched) {   // the gather ran on the comm stream (tt_contract_prefetch)
    TT_CUDA(cudaStreamWaitEvent(ctx->stream, pl->pf_event, 0));
    pl->prefetched = false;
  } else {
    TT_TRY(run_gather(ctx, pl->gp, A == B ? std::vector<tt_tensor>{A} : std::vector<tt_tensor>{A, B}));
  }
  // measured autotuning (large plans, TT_AUTOTUNE != 0): the first call times the model's variant, the
  // second the runner-up, later calls use the faster (> 1 % better).  Every variant accumulates each
  // output element over the same k sequence, so the choice never changes the result bits (R12;
  // tests/test_gpu_parity.py::test_variants_bitwise_equal).  Not inside stream capture.
  const ContractPlan* run = pl.get();
  static const bool autotune = [] { const char* e = getenv("TT_AUTOTUNE"); return !e || atoi(e) != 0; }();
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  TT_CUDA(cudaStreamIsCapturing(ctx->stream, &cap));
  const bool tuning = autotune && pl->tune < 2 && pl->alt_variant >= 0 && pl->variant >= num_contract_variants() &&
                      pl->flops >= 5e10 &&
                      cap == cudaStreamCaptureStatusNone && !getenv("TT_FORCE_VARIANT");
  if (tuning && pl->tune == 1 && !pl->alt) {
    ContractOpts o;
    o.force_variant = pl->alt_variant;
    o.tag = "|alt";
    TT_TRY(get_contract_plan(ctx, C, cl, A, al, B, bl, beta, pl->alt, nullptr, o));
  }
  if (pl->tune == 2 && pl->use_alt) run = pl->alt.get();
  if (tuning) {
    if (pl->tune == 1) run = pl->alt.get();
    cudaEvent_t e0, e1;
    TT_CUDA(cudaEventCreate(&e0));
    TT_CUDA(cudaEventCreate(&e1));
    TT_CUDA(cudaEventRecord(e0, ctx->stream));
    TT_TRY(launch_plan(ctx, *run, C, cl, beta, alpha, A, al, B, bl));
    TT_CUDA(cudaEventRecord(e1, ctx->stream));
    TT_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    TT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (pl->tune == 0) {
      pl->tune_ms = ms;
      pl->tune = 1;
    } else {
      pl->use_alt = ms < 0.99f * pl->tune_ms;
      pl->tune = 2;
    }
  } else {
    TT_TRY(launch_plan(ctx, *run, C, cl, beta, alpha, A, al, B, bl));
  }
  ctx->last.c_blocks = (int64_t)pl->my.size();
  ctx->last.tasks = pl->tasks;
  ctx->last.work_items = pl->nwork;
  ctx->last.flops = pl->flops;
  ctx->last.bytes = pl->bytes;
  ctx->last.gathered_bytes = pl->gp.recv_bytes;
  ctx->last.plan_cached = was_cached ? 1 : 0;
  ctx->last.kernel_variant = run->variant;
  ctx->last.producer = run->tma ? 1 : 0;
  return TT_OK;
}

tt_status tt_contract_prefetch(tt_ctx ctx, tt_tensor C, const char* cl, double beta, tt_tensor A, const char* al,
                               tt_tensor B, const char* bl) {
  NvtxRange nvtx_("tt_contract_prefetch");
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  std::shared_ptr<ContractPlan> pl;
  TT_TRY(get_contract_plan(ctx, C, cl, A, al, B, bl, beta, pl, nullptr));
  TT_TRY(need_ws(ctx));
  if (ctx->prepare_only || ctx->nranks <= 1) return TT_OK;
  TT_TRY(check_bound(A, "A"));
  TT_TRY(check_bound(B, "B"));
  if (pl->prefetched) return fail(TT_E_STATE, "this contraction's gather is already prefetched");
  DeviceGuard dg(ctx->device);
  if (!ctx->comm_stream) {
    TT_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    TT_CUDA(cudaEventCreateWithFlags(&ctx->comm_fork, cudaEventDisableTiming));
    TT_CUDA(cudaEventCreateWithFlags(&ctx->comm_done, cudaEventDisableTiming));
  }
  if (!pl->pf_event) TT_CUDA(cudaEventCreateWithFlags(&pl->pf_event, cudaEventDisableTiming));
  // the gather overwrites non-owned input ranges: it starts after everything issued on the context
  // stream so far (no write-after-read hazard with earlier kernels), and the consuming tt_contract waits
  TT_CUDA(cudaEventRecord(ctx->comm_fork, ctx->stream));
  TT_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->comm_fork, 0));
  TT_TRY(run_gather(ctx, pl->gp, A == B ? std::vector<tt_tensor>{A} : std::vector<tt_tensor>{A, B}, ctx->comm_stream));
  TT_CUDA(cudaEventRecord(pl->pf_event, ctx->comm_stream));
  TT_CUDA(cudaEventRecord(ctx->comm_done, ctx->comm_stream));
  ctx->comm_pending = true;
  pl->prefetched = true;
  return TT_OK;
}

// End to end from host memory (tt.h tt_contract_host).  Pipelined (nranks == 1, A's and C's dim 0 carry
// the same label on the same tiling, no views): per dim-0 tile x of C, A's blocks with dim-0 coordinate x
// -- one contiguous packed range (row-major block order) -- go host->device on the context's copy stream
// while tile x-1 contracts; tile x is a local plan restricted to C's blocks with dim-0 coordinate x (the
// same kernel and per-element k order as the whole contraction: bitwise the same result, R12); its C
// rows go device->host while tile x+1 contracts.  Otherwise: H2D of every held range, tt_contract, D2H
// of this rank's C ranges.
namespace {
struct HostPlan {
  bool pipelined = false;
  std::vector<std::pair<int64_t, int64_t>> a_rng, c_rng;   // per dim-0 tile of C: storage ranges of A, C
  std::vector<std::shared_ptr<ContractPlan>> tiles;        // local plan of each tile (nullptr: no C block)
};

void held_storage(tt_tensor T, int32_t rank, std::vector<std::pair<int64_t, int64_t>>& out) {
  out.clear();
  std::vector<std::pair<int64_t, int64_t>> hr;
  for (int64_t b = 0; b < T->nblocks; ++b) {
    if (!T->nz[b] || T->blk_off[b] < 0) continue;
    T->held_ranges(b, rank, hr);
    for (auto& h : hr) {
      const int64_t a0 = T->blk_off[b] + h.first, a1 = T->blk_off[b] + h.second;
      if (!out.empty() && a0 - out.back().second <= 1) out.back().second = std::max(out.back().second, a1);
      else out.push_back({a0, a1});
    }
  }
}

tt_status h2d(tt_tensor T, const double* h, const std::vector<std::pair<int64_t, int64_t>>& rng, cudaStream_t st) {
  for (auto& r : rng)
    if (r.second > r.first)
      TT_CUDA(cudaMemcpyAsync(T->data + r.first, h + r.first, (r.second - r.first) * 8, cudaMemcpyHostToDevice, st));
  return TT_OK;
}
tt_status d2h(tt_tensor T, double* h, const std::vector<std::pair<int64_t, int64_t>>& rng, cudaStream_t st) {
  for (auto& r : rng)
    if (r.second > r.first)
      TT_CUDA(cudaMemcpyAsync(h + r.first, T->data + r.first, (r.second - r.first) * 8, cudaMemcpyDeviceToHost, st));
  return TT_OK;
}
}  // namespace

tt_status tt_contract_host(tt_ctx ctx, tt_tensor C, const char* cl, double beta, double alpha, tt_tensor A,
                           const char* al, tt_tensor B, const char* bl, const double* hA, const double* hB, double* hC,
                           int32_t c_flags) {
  NvtxRange nvtx_("tt_contract_host");
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  if ((c_flags & ~(TT_HOST_C_IN | TT_HOST_C_OUT)) != 0) return fail(TT_E_ARG, "unknown c_flags bits");
  if ((c_flags & (TT_HOST_C_IN | TT_HOST_C_OUT)) && !hC) return fail(TT_E_ARG, "c_flags name C but hC is NULL");
  std::shared_ptr<ContractPlan> whole;
  TT_TRY(get_contract_plan(ctx, C, cl, A, al, B, bl, beta, whole, nullptr));
  TT_TRY(need_ws(ctx));
  TT_TRY(check_bound(C, "C"));
  TT_TRY(check_bound(A, "A"));
  TT_TRY(check_bound(B, "B"));
  DeviceGuard dg(ctx->device);
  const std::string key = plan_key("host", C, cl, A, al, B, bl, beta);
  auto hp = cached<HostPlan>(ctx, key);
  if (!hp) {
    hp = std::make_shared<HostPlan>();
    const bool same0 = al[0] == cl[0] && same_tiling(A->dims[0], C->dims[0]);
    hp->pipelined = ctx->nranks == 1 && same0 && !A->view_of && !C->view_of && A != B && !C->compact;
    if (hp->pipelined) {
      const int32_t nt = C->dims[0]->ntiles();
      hp->a_rng.assign(nt, {0, 0});
      hp->c_rng.assign(nt, {0, 0});
      hp->tiles.assign(nt, nullptr);
      int32_t co[TT_MAX_ORDER];
      auto span = [&](tt_tensor T, std::vector<std::pair<int64_t, int64_t>>& rng) {
        for (int64_t b = 0; b < T->nblocks; ++b) {
          if (!T->nz[b] || T->blk_off[b] < 0) continue;
          T->block_coords(b, co);
          auto& r = rng[co[0]];
          const int64_t a0 = T->blk_off[b], a1 = a0 + T->block_volume(b);
          if (r.second == r.first) r = {a0, a1};
          else r = {std::min(r.first, a0), std::max(r.second, a1)};
        }
      };
      span(A, hp->a_rng);
      span(C, hp->c_rng);
      for (int32_t x = 0; x < nt; ++x) {
        ContractOpts o;
        o.local = true;
        o.tag = "|host" + std::to_string(x);
        for (int64_t b = 0; b < C->nblocks; ++b) {
          if (!C->nz[b]) continue;
          C->block_coords(b, co);
          if (co[0] == x) o.sel.push_back({b, 0, C->ext0(b)});
        }
        if (o.sel.empty()) continue;
        TT_TRY(get_contract_plan(ctx, C, cl, A, al, B, bl, beta, hp->tiles[x], nullptr, o));
      }
    }
    plan_put(ctx, key, hp);
  }
  std::vector<std::pair<int64_t, int64_t>> rB, rC, rA;
  if (hB) held_storage(B, ctx->rank, rB);
  if (hC) held_storage(C, ctx->rank, rC);
  if (!hp->pipelined || !hA) {
    if (hA) {
      held_storage(A, ctx->rank, rA);
      TT_TRY(h2d(A, hA, rA, ctx->stream));
    }
    if (hB) TT_TRY(h2d(B, hB, rB, ctx->stream));
    if (c_flags & TT_HOST_C_IN) TT_TRY(h2d(C, hC, rC, ctx->stream));
    TT_TRY(tt_contract(ctx, C, cl, beta, alpha, A, al, B, bl));
    if (c_flags & TT_HOST_C_OUT) TT_TRY(d2h(C, hC, rC, ctx->stream));
    return TT_OK;
  }
  if (!ctx->copy_stream) {
    TT_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    TT_CUDA(cudaEventCreateWithFlags(&ctx->copy_fork, cudaEventDisableTiming));
  }
  const int32_t nt = (int32_t)hp->tiles.size();
  while ((int32_t)ctx->tile_events.size() < 2 * nt + 1) {
    cudaEvent_t e;
    TT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->tile_events.push_back(e);
  }
  cudaEvent_t* up = ctx->tile_events.data();          // A rows of tile x arrived
  cudaEvent_t* done = up + nt;                        // tile x contracted
  cudaEvent_t fin = ctx->tile_events[2 * nt];
  // B and the incoming C on the context stream; A tile by tile on the copy stream, after everything
  // already queued on the context stream (no overwrite of data earlier kernels still read)
  if (hB) TT_TRY(h2d(B, hB, rB, ctx->stream));
  if (c_flags & TT_HOST_C_IN) TT_TRY(h2d(C, hC, rC, ctx->stream));
  TT_CUDA(cudaEventRecord(ctx->copy_fork, ctx->stream));
  TT_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_fork, 0));
  for (int32_t x = 0; x < nt; ++x) {
    TT_TRY(h2d(A, hA, {hp->a_rng[x]}, ctx->copy_stream));
    TT_CUDA(cudaEventRecord(up[x], ctx->copy_stream));
  }
  reset_stats(ctx);
  double flops = 0;
  int64_t tasks = 0;
  for (int32_t x = 0; x < nt; ++x) {
    TT_CUDA(cudaStreamWaitEvent(ctx->stream, up[x], 0));
    if (hp->tiles[x]) {
      TT_TRY(launch_plan(ctx, *hp->tiles[x], C, cl, beta, alpha, A, al, B, bl));
      flops += hp->tiles[x]->flops;
      tasks += hp->tiles[x]->tasks;
    }
    TT_CUDA(cudaEventRecord(done[x], ctx->stream));
  }
  if (c_flags & TT_HOST_C_OUT)
    for (int32_t x = 0; x < nt; ++x) {
      TT_CUDA(cudaStreamWaitEvent(ctx->copy_stream, done[x], 0));
      TT_TRY(d2h(C, hC, {hp->c_rng[x]}, ctx->copy_stream));
    }
  TT_CUDA(cudaEventRecord(fin, ctx->copy_stream));
  TT_CUDA(cudaStreamWaitEvent(ctx->stream, fin, 0));
  ctx->last.flops = flops;
  ctx->last.tasks = tasks;
  ctx->last.bytes = whole->bytes;
  return TT_OK;
}

tt_status tt_task_list(tt_ctx ctx, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                       const char* bl, int32_t where, int64_t* cblk, int64_t* ptr, int64_t* a_blk, int64_t* b_blk,
                       int64_t* cost, int64_t cap, int64_t* n_cblocks, int64_t* n_tasks) {
  if (!ctx || !n_cblocks || !n_tasks) return fail(TT_E_ARG, "NULL argument");
  Analysis an;
  TT_TRY(analyse(C, cl, A, al, B, bl, an));
  if (where == 0) {
    HostTasks ht;
    enumerate_tasks(an, C, A, B, ht);
    *n_cblocks = (int64_t)ht.cblk.size();
    *n_tasks = (int64_t)ht.a_blk.size();
    if (!a_blk) return TT_OK;
    if (cap < *n_tasks) return fail(TT_E_ARG, "capacity %lld < %lld tasks", (long long)cap, (long long)*n_tasks);
    std::copy(ht.cblk.begin(), ht.cblk.end(), cblk);
    std::copy(ht.ptr.begin(), ht.ptr.end(), ptr);
    std::copy(ht.a_blk.begin(), ht.a_blk.end(), a_blk);
    std::copy(ht.b_blk.begin(), ht.b_blk.end(), b_blk);
    if (cost) std::copy(ht.cost.begin(), ht.cost.end(), cost);
    return TT_OK;
  }
  TT_TRY(need_ws(ctx));
  std::shared_ptr<ContractPlan> pl;
  TT_TRY(get_contract_plan(ctx, C, cl, A, al, B, bl, 1.0, pl, nullptr));
  const HostTasks& ht = pl->ht;
  *n_cblocks = (int64_t)ht.cblk.size();
  *n_tasks = (int64_t)ht.a_blk.size();
  if (!a_blk) return TT_OK;
  if (cap < *n_tasks) return fail(TT_E_ARG, "capacity %lld < %lld tasks", (long long)cap, (long long)*n_tasks);
  DeviceGuard dg(ctx->device);
  // device-built arrays (ptr, a_blk, b_blk) copied back; cblk / cost are host plan metadata
  std::copy(ht.cblk.begin(), ht.cblk.end(), cblk);
  TT_CUDA(cudaMemcpy(ptr, pl->d_ptr, (*n_cblocks + 1) * 8, cudaMemcpyDeviceToHost));
  if (*n_tasks) {
    TT_CUDA(cudaMemcpy(a_blk, pl->d_ablk, *n_tasks * 8, cudaMemcpyDeviceToHost));
    TT_CUDA(cudaMemcpy(b_blk, pl->d_bblk, *n_tasks * 8, cudaMemcpyDeviceToHost));
  }
  if (cost) std::copy(ht.cost.begin(), ht.cost.end(), cost);
  return TT_OK;
}

tt_status tt_partition_lpt(tt_ctx ctx, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                           const char* bl, uint32_t group_mask, int32_t* owner) {
  if (!ctx || !owner) return fail(TT_E_ARG, "NULL argument");
  Analysis an;
  TT_TRY(analyse(C, cl, A, al, B, bl, an));
  if (group_mask >> C->order) return fail(TT_E_ARG, "group_mask references dims beyond the order of C");
  HostTasks ht;
  enumerate_tasks(an, C, A, B, ht);
  // units: blocks sharing the tile coordinates of the grouping dims (group_mask = 0: single blocks)
  std::map<std::vector<int32_t>, size_t> unit_of;
  std::vector<int64_t> ucost, uid;
  std::vector<size_t> unit(ht.cblk.size());
  int32_t cc[TT_MAX_ORDER];
  for (size_t g = 0; g < ht.cblk.size(); ++g) {
    std::vector<int32_t> key;
    if (group_mask) {
      C->block_coords(ht.cblk[g], cc);
      for (int d = 0; d < C->order; ++d)
        if (group_mask >> d & 1) key.push_back(cc[d]);
    } else {
      key.push_back((int32_t)g);
    }
    auto it = unit_of.find(key);
    if (it == unit_of.end()) {
      it = unit_of.emplace(key, ucost.size()).first;
      ucost.push_back(0);
      uid.push_back(ht.cblk[g]);      // smallest block id of the unit (blocks visited in order)
    }
    unit[g] = it->second;
    ucost[it->second] += ht.cost[g];
  }
  std::vector<int32_t> own = lpt(ucost, uid, ctx->nranks);
  for (int64_t b = 0; b < C->nblocks; ++b) owner[b] = -1;
  for (size_t g = 0; g < ht.cblk.size(); ++g) owner[ht.cblk[g]] = own[unit[g]];
  return TT_OK;
}

namespace {
// water-filling partition with row splitting over (non-zero C block, cost) pairs in block order
tt_status split_partition(tt_ctx ctx, tt_tensor C, const std::vector<int64_t>& cblk,
                          const std::vector<int64_t>& cost, uint32_t group_mask) {
  if (C->view_of) return fail(TT_E_UNSUPPORTED, "a view takes its owners from its parent");
  TT_TRY(check_no_views(C));
  if (group_mask >> C->order) return fail(TT_E_ARG, "group_mask references dims beyond the order of C");
  if (group_mask && !(group_mask & 1u)) return fail(TT_E_ARG, "row splitting needs dim 0 among the grouping dims");
  // units (as tt_partition_lpt)
  std::map<std::vector<int32_t>, size_t> unit_of;
  std::vector<int64_t> ucost, uid, urows;
  std::vector<std::vector<int64_t>> ublocks;
  int32_t cc[TT_MAX_ORDER];
  for (size_t g = 0; g < cblk.size(); ++g) {
    std::vector<int32_t> key;
    C->block_coords(cblk[g], cc);
    if (group_mask) {
      for (int d = 0; d < C->order; ++d)
        if (group_mask >> d & 1) key.push_back(cc[d]);
    } else {
      key.push_back((int32_t)g);
    }
    auto it = unit_of.find(key);
    if (it == unit_of.end()) {
      it = unit_of.emplace(key, ucost.size()).first;
      ucost.push_back(0);
      uid.push_back(cblk[g]);
      urows.push_back(C->dims[0]->size(cc[0]));
      ublocks.push_back({});
    }
    ucost[it->second] += cost[g];
    ublocks[it->second].push_back(cblk[g]);
  }
  std::vector<size_t> order(ucost.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
    if (ucost[x] != ucost[y]) return ucost[x] > ucost[y];
    return uid[x] < uid[y];
  });
  // water-filling along the ordered cost axis: rank r owns [B_r, B_{r+1}), B_r = floor(r*W/P);
  // a unit straddling a boundary is cut at the nearest row (round half up)
  const int P = ctx->nranks;
  __int128 W = 0;
  for (int64_t c : ucost) W += c;
  std::vector<int64_t> Bd(P + 1);
  for (int r = 0; r <= P; ++r) Bd[r] = (int64_t)((__int128)r * W / P);
  std::vector<int32_t> own(C->nblocks, -1);
  std::vector<std::vector<tt_tensor_s::Part>> parts(C->nblocks);
  int64_t cum = 0;
  for (size_t u : order) {
    const int64_t c0 = cum, c1 = cum + ucost[u], rows = urows[u];
    cum = c1;
    int r0 = 0;
    for (int r = 1; r < P; ++r)
      if (Bd[r] <= c0) r0 = r;
    std::vector<tt_tensor_s::Part> pp;
    int cur = r0;
    int64_t start = 0;
    for (int r = r0 + 1; r < P && ucost[u] > 0; ++r) {
      if (Bd[r] >= c1) break;
      int64_t row = (int64_t)(((__int128)(Bd[r] - c0) * rows * 2 + ucost[u]) / ((__int128)2 * ucost[u]));
      row = std::min(std::max(row, (int64_t)0), rows);
      if (row > start) {
        pp.push_back({(int32_t)start, (int32_t)row, cur});
        start = row;
      }
      cur = r;
    }
    if (rows > start) pp.push_back({(int32_t)start, (int32_t)rows, cur});
    for (int64_t b : ublocks[u]) {
      if (pp.size() == 1) own[b] = pp[0].owner;
      else { own[b] = TT_SPLIT; parts[b] = pp; }
    }
  }
  for (int64_t b = 0; b < C->nblocks; ++b) C->owner[b] = C->nz[b] ? own[b] : -1;
  C->parts = parts;
  refresh_parts_view(C);
  apply_storage(C);
  C->version++;
  return TT_OK;
}
}  // namespace

tt_status tt_partition_split(tt_ctx ctx, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                             const char* bl, uint32_t group_mask) {
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  Analysis an;
  TT_TRY(analyse(C, cl, A, al, B, bl, an));
  HostTasks ht;
  enumerate_tasks(an, C, A, B, ht);
  return split_partition(ctx, C, ht.cblk, ht.cost, group_mask);
}

tt_status tt_partition_split_cost(tt_ctx ctx, tt_tensor C, const int64_t* cost, uint32_t group_mask) {
  if (!ctx || !C || !cost) return fail(TT_E_ARG, "NULL context, tensor or cost array");
  std::vector<int64_t> cblk, cst;
  for (int64_t b = 0; b < C->nblocks; ++b) {
    if (!C->nz[b]) continue;
    const int64_t c = cost[cblk.size()];
    if (c < 0) return fail(TT_E_ARG, "negative block cost");
    cblk.push_back(b);
    cst.push_back(c);
  }
  return split_partition(ctx, C, cblk, cst, group_mask);
}

}  // extern "C"

namespace {   // defined with tt_contract_cholesky below
void chol_maps(tt_tensor X, const std::vector<tt_tis>& vd, std::vector<uint8_t>& vnz, std::vector<uint8_t>& wnz);
tt_status chol_check(tt_tensor C, const char* cl, tt_tensor X, const char* vl, tt_tensor B, const char* bl,
                     std::vector<tt_tis>& vd);
tt_status new_meta_tensor(tt_ctx ctx, const std::vector<tt_tis>& dims, const std::vector<uint8_t>& nz, tt_tensor* out);
}  // namespace

extern "C" {

tt_status tt_partition_split_cholesky(tt_ctx ctx, tt_tensor C, const char* cl, tt_tensor X, const char* vl,
                                      tt_tensor B, const char* bl, uint32_t group_mask) {
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  std::vector<tt_tis> vd;
  TT_TRY(chol_check(C, cl, X, vl, B, bl, vd));
  std::vector<uint8_t> vnz, wnz;
  chol_maps(X, vd, vnz, wnz);
  tt_tensor W = nullptr;
  TT_TRY(new_meta_tensor(ctx, vd, wnz, &W));
  std::unique_ptr<tt_tensor_s> hold(W);
  Analysis an;
  TT_TRY(analyse(C, cl, W, vl, B, bl, an));
  HostTasks ht;
  enumerate_tasks(an, C, W, B, ht);
  // W formation of one (p_t, q_t) row: 2 N_L |p||q| sum over W's (r_t, s_t) blocks of |r||s|, shared
  // evenly (integer division) by the row's non-zero C blocks
  const std::string c(cl);
  const int pc = (int)c.find(vl[0]), qc = (int)c.find(vl[1]);
  const int64_t NL = X->dims[2]->offsets.back();
  const int32_t np = vd[0]->ntiles(), nq = vd[1]->ntiles(), nr = vd[2]->ntiles(), ns = vd[3]->ntiles();
  std::vector<int64_t> build((size_t)np * nq, 0), cnt((size_t)np * nq, 0), row(ht.cblk.size());
  for (int32_t a = 0; a < np; ++a)
    for (int32_t bq = 0; bq < nq; ++bq) {
      int64_t w = 0;
      for (int32_t r = 0; r < nr; ++r)
        for (int32_t s = 0; s < ns; ++s)
          if (wnz[(((int64_t)a * nq + bq) * nr + r) * ns + s]) w += vd[2]->size(r) * vd[3]->size(s);
      build[(size_t)a * nq + bq] = 2 * NL * vd[0]->size(a) * vd[1]->size(bq) * w;
    }
  int32_t cc[TT_MAX_ORDER];
  for (size_t g = 0; g < ht.cblk.size(); ++g) {
    C->block_coords(ht.cblk[g], cc);
    row[g] = (int64_t)cc[pc] * nq + cc[qc];
    cnt[row[g]]++;
  }
  std::vector<int64_t> cost(ht.cblk.size());
  for (size_t g = 0; g < ht.cblk.size(); ++g) cost[g] = ht.cost[g] + build[row[g]] / std::max<int64_t>(cnt[row[g]], 1);
  return split_partition(ctx, C, ht.cblk, cost, group_mask);
}

tt_status tt_gather_plan(tt_ctx ctx, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                         const char* bl, int64_t* recv, int64_t* n_recv, int64_t* send, int64_t* n_send, int64_t cap) {
  if (!ctx || !n_recv || !n_send) return fail(TT_E_ARG, "NULL argument");
  Analysis an;
  TT_TRY(analyse(C, cl, A, al, B, bl, an));
  if (C == A || C == B) return fail(TT_E_ARG, "C must not alias A or B");
  ContractPlan pl;
  pl.an = an;
  tt_ctx_s host;             // host-only planning context (no device work)
  host.device = -1;
  host.rank = ctx->rank;
  host.nranks = ctx->nranks;
  host.sm_count = ctx->sm_count;
  TT_TRY(build_contract_plan(&host, C, A, B, 1.0, pl));
  *n_recv = (int64_t)pl.gp.recv_list.size() / 5;
  *n_send = (int64_t)pl.gp.send_list.size() / 5;
  if (!recv && !send) return TT_OK;
  if (cap < std::max(*n_recv, *n_send)) return fail(TT_E_ARG, "capacity too small");
  if (recv) std::copy(pl.gp.recv_list.begin(), pl.gp.recv_list.end(), recv);
  if (send) std::copy(pl.gp.send_list.begin(), pl.gp.send_list.end(), send);
  return TT_OK;
}

}  // extern "C"

// =============================================================================================
// Implicit Cholesky-factored operand (PAPER Eq. cc12, P312-318)
//
//   C(c) = beta*C + alpha * sum_{r,s} V(p,q,r,s) * B(..r..s..)   with V never stored:
//   V(p,q,r,s) = W(p,q,r,s) - W(p,q,s,r),   W(p,q,r,s) = sum_L X(p,r,L) X(q,s,L)   (Eq. cc12, R19)
//
// Because the exchange term of Eq. cc12 is the Coulomb term W with r and s swapped, re-indexing the
// second sum gives exactly
//   sum_{r,s} V(p,q,r,s) B(..r..s..) = sum_{r,s} W(p,q,r,s) Bm(..r..s..),  Bm = B - B(r<->s)
// so only the Coulomb blocks W are built (one DMMA contraction over L per block).  Bm is
// antisymmetric in (r,s), so only its tile pairs r_t <= s_t are formed ("Bh", about half of B):
//   sum_{r,s} W Bm = sum_{r_t <= s_t} W(p,q,r,s) Bh(r,s) - sum_{r_t < s_t} W(p,q,s,r) Bh(r,s)
// (pass 1 over Bh's blocks, pass 2 over its strictly-upper blocks with W read as (p,q,s,r)): the
// same consume FLOPs as a full Bm, half its memory.  When B's blocks (r,s) and (s,r) sit on the same
// rank, each rank forms its own Bh blocks from its own B blocks and Bh is all-gathered (half of B's
// bytes; B itself may then use compact storage); otherwise B is all-gathered and every rank forms
// all of Bh.  The rank's C parts are processed in batches of (p,q) tile rows: W of the batch is
// built into the workspace and immediately consumed restricted to the batch.  X must be replicated.
// When the workspace cannot hold Bh plus one W row (or TT_CHOL_TWO_PASS=1) the consume reads B
// directly in two passes, C += alpha W.B and C -= alpha W.B(r<->s): no Bh, twice the consume FLOPs.

namespace {

// TT_DEBUG=1: phase trace of the implicit-operand driver on stderr (synchronises the stream)
struct PhaseTrace {
  tt_ctx ctx;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseTrace(tt_ctx c) : ctx(c), on(getenv("TT_DEBUG") && atoi(getenv("TT_DEBUG")) != 0),
                                  t0(std::chrono::steady_clock::now()) {}
  void operator()(const char* what, long long a = -1) {
    if (!on) return;
    cudaStreamSynchronize(ctx->stream);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[tt rank %d] %10.1f ms  %s %lld\n", ctx->rank, ms, what, a);
    fflush(stderr);
  }
};

struct CholBatch {
  tt_tensor Wb = nullptr;            // scratch W blocks of the batch (bound to the workspace)
  ContractOpts wopt, copt;           // local build / consume selections
};

struct CholPlan {
  tt_tensor Vmeta = nullptr, Wmeta = nullptr;   // block maps of V (algorithmic count) and W
  tt_tensor Bh = nullptr;                       // (B - B(r<->s)) on tile pairs r_t <= s_t, in the workspace
  tt_tensor Bs = nullptr;                       // view of Bh's strictly-upper blocks (r_t < s_t)
  std::shared_ptr<ContractPlan> vplan, wplan;   // SPMD plans: this rank's C parts, FLOP counts
  std::shared_ptr<ElemPlan> copy_plan, swap_plan;   // Bh formation (this rank's Bh blocks)
  GatherPlan bgather;                           // all-gather of B (not co-located) ...
  GatherPlan hgather;                           // ... or of Bh (co-located B pairs)
  std::vector<CholBatch> batches;
  std::string lc;                               // the auxiliary label used for L
  bool two_pass = false;                        // no room for Bh: consume W.B and W.B(r<->s)
  bool colocated = false;
  ~CholPlan() {
    delete Vmeta;
    delete Wmeta;
    delete Bh;
    delete Bs;
    for (auto& b : batches) delete b.Wb;
  }
};

tt_status new_meta_tensor(tt_ctx ctx, const std::vector<tt_tis>& dims, const std::vector<uint8_t>& nz, tt_tensor* out) {
  tt_tensor t;
  TT_TRY(tensor_new(ctx, (int32_t)dims.size(), dims.data(), &t));
  t->nz = nz;
  tensor_finish(t);
  *out = t;
  return TT_OK;
}

// local element add X(all blocks) = beta*X + alpha*Y(perm) with no gather (Y fully present)
tt_status local_add_plan(tt_ctx ctx, tt_tensor Xt, tt_tensor Yt, const std::vector<int>& perm, double beta,
                         std::shared_ptr<ElemPlan>& out, const std::vector<uint8_t>* only = nullptr) {
  auto ep = std::make_shared<ElemPlan>();
  int32_t cc[TT_MAX_ORDER], ac[TT_MAX_ORDER];
  for (int64_t b = 0; b < Xt->nblocks; ++b) {
    if (!Xt->nz[b] || (only && !(*only)[b])) continue;
    Xt->block_coords(b, cc);
    for (int d = 0; d < Xt->order; ++d) ac[perm[d]] = cc[d];
    const int64_t ab = Yt->block_id(ac);
    ElemDesc d{};
    d.x_off = Xt->blk_off[b];
    d.y_off = Yt->nz[ab] ? Yt->blk_off[ab] : -1;
    int64_t sa[TT_MAX_ORDER], acc = 1;
    for (int q = Yt->order - 1; q >= 0; --q) { sa[q] = acc; acc *= Yt->dims[q]->size(ac[q]); }
    int32_t ext[TT_MAX_ORDER];
    for (int q = 0; q < Xt->order; ++q) ext[q] = (int32_t)Xt->dims[q]->size(cc[q]);
    fuse_elem(d, Xt->order, ext, perm.data(), sa);
    emit_elem(*ep, d, true, {{0, Xt->block_volume(b)}});
    ep->bytes += 8.0 * Xt->block_volume(b) * ((beta != 0.0) + 2);
    ep->blocks++;
  }
  TT_TRY(upload_elem(ctx, *ep, false));
  out = ep;
  return TT_OK;
}

// Block maps of the implicit operand over its tiled spaces vd = (p, q, r, s) (reading R19b): from X's
// (p_t, r_t) tile pairs holding any non-zero block (over all L tiles) -- X's actual block map, not the
// tiles' spins.  W(pqrs) = sum_L X(prL) X(qsL) (the Coulomb term) is non-zero where both factors are;
// V = W - W(r<->s) where the Coulomb or the exchange term is.
void chol_maps(tt_tensor X, const std::vector<tt_tis>& vd, std::vector<uint8_t>& vnz, std::vector<uint8_t>& wnz) {
  int64_t nvb = 1;
  for (auto t : vd) nvb *= t->ntiles();
  const int32_t nx0 = X->grid[0], nx1 = X->grid[1];
  std::vector<uint8_t> xnz((size_t)nx0 * nx1, 0);
  int32_t xc[TT_MAX_ORDER];
  for (int64_t xb = 0; xb < X->nblocks; ++xb)
    if (X->nz[xb]) {
      X->block_coords(xb, xc);
      xnz[(size_t)xc[0] * nx1 + xc[1]] = 1;
    }
  vnz.assign(nvb, 0);
  wnz.assign(nvb, 0);
  for (int64_t x = 0; x < nvb; ++x) {
    int64_t y = x;
    int32_t co[4];
    for (int d = 3; d >= 0; --d) { co[d] = (int32_t)(y % vd[d]->ntiles()); y /= vd[d]->ntiles(); }
    auto xn = [&](int32_t u, int32_t w) { return xnz[(size_t)u * nx1 + w] != 0; };
    wnz[x] = (xn(co[0], co[2]) && xn(co[1], co[3])) ? 1 : 0;              // Coulomb term reachable
    vnz[x] = (wnz[x] || (xn(co[0], co[3]) && xn(co[1], co[2]))) ? 1 : 0;  // Coulomb or exchange
  }
}

// Shared validation of the implicit-operand ladder C(..p..q..) += V(p,q,r,s) B(..r..s..) (Eq. cc12):
// labels, ladder form and tilings; returns the four tiled spaces and the labels.
tt_status chol_check(tt_tensor C, const char* cl, tt_tensor X, const char* vl, tt_tensor B, const char* bl,
                     std::vector<tt_tis>& vd) {
  if (!C || !X || !B || !vl) return fail(TT_E_ARG, "NULL argument");
  TT_TRY(check_labels(cl, C, "C"));
  TT_TRY(check_labels(bl, B, "B"));
  const std::string c(cl), v(vl), b(bl);
  if (v.size() != 4) return fail(TT_E_LABEL, "the implicit operand V(p,q,r,s) needs 4 labels");
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j)
      if (v[i] == v[j]) return fail(TT_E_LABEL, "repeated label in V");
  if (X->order != 3) return fail(TT_E_ARG, "X must be order 3: X(p, r, L)");
  const char p = v[0], q = v[1], r = v[2], s = v[3];
  if (c.find(p) == std::string::npos || c.find(q) == std::string::npos)
    return fail(TT_E_UNSUPPORTED, "V's first two labels must be free labels of C (ladder form)");
  if (b.find(r) == std::string::npos || b.find(s) == std::string::npos || c.find(r) != std::string::npos ||
      c.find(s) != std::string::npos)
    return fail(TT_E_UNSUPPORTED, "V's last two labels must be contracted with B (ladder form)");
  vd = {C->dims[c.find(p)], C->dims[c.find(q)], B->dims[b.find(r)], B->dims[b.find(s)]};
  for (tt_tis t : vd)
    if (!same_tiling(t, X->dims[0]) || !same_tiling(t, X->dims[1]))
      return fail(TT_E_TILING, "V's labels and X's first two dims must share one tiled space (Eq. cc12)");
  return TT_OK;
}

tt_status run_local_add(tt_ctx ctx, const ElemPlan& ep, tt_tensor Xt, tt_tensor Yt, double beta, double alpha) {
  ElemParams p{};
  p.X = Xt->data;
  p.Y = Yt->data;
  p.descs = ep.d_descs;
  p.segs = ep.d_segs;
  p.tiles = ep.d_tiles;
  p.order = Xt->order;
  p.alpha = alpha;
  p.beta = beta;
  Launch L(ctx, "tt_add[cholesky Bh]");
  TT_CUDA(launch_add(p, ep.nseg(), ep.ntiles(), ctx->stream));
  return TT_OK;
}

}  // namespace

extern "C" {

tt_status tt_contract_cholesky(tt_ctx ctx, tt_tensor C, const char* cl, double beta, double alpha, tt_tensor X,
                               const char* vl, tt_tensor B, const char* bl, void* workspace, int64_t ws_elems) {
  NvtxRange nvtx_("tt_contract_cholesky");
  if (!ctx) return fail(TT_E_ARG, "NULL context");
  std::vector<tt_tis> vdims;
  TT_TRY(chol_check(C, cl, X, vl, B, bl, vdims));
  const std::string c(cl), v(vl), b(bl);
  const char p = v[0], q = v[1], r = v[2], s = v[3];
  tt_tis tp = vdims[0], tq = vdims[1], tr = vdims[2], ts = vdims[3];
  if (ctx->nranks > 1)
    for (int64_t x = 0; x < X->nblocks; ++x)
      if (X->nz[x] && X->owner[x] != TT_REPLICATED)
        return fail(TT_E_UNSUPPORTED, "with nranks > 1 the Cholesky vectors X must be replicated");
  std::string lc;
  for (char ch : std::string("LMNOPQRSTUVWXYZ0123456789"))
    if (c.find(ch) == std::string::npos && v.find(ch) == std::string::npos && b.find(ch) == std::string::npos) {
      lc = std::string(1, ch);
      break;
    }
  TT_TRY(need_ws(ctx));
  TT_TRY(check_bound(C, "C"));
  TT_TRY(check_bound(X, "X"));
  TT_TRY(check_bound(B, "B"));
  if (!workspace || ws_elems <= 0) return fail(TT_E_UNBOUND, "no workspace bound");
  DeviceGuard dg(ctx->device);
  PhaseTrace trace(ctx);

  char keybuf[256];
  snprintf(keybuf, sizeof(keybuf), "chol|%llu.%llu|%llu.%llu|%llu.%llu|%s|%s|%s|%d|%p|%lld",
           (unsigned long long)C->uid, (unsigned long long)C->version, (unsigned long long)X->uid,
           (unsigned long long)X->version, (unsigned long long)B->uid, (unsigned long long)B->version, cl, vl, bl,
           beta != 0.0, workspace, (long long)ws_elems);
  auto cp = cached<CholPlan>(ctx, keybuf);
  if (!cp) {
    cp = std::make_shared<CholPlan>();
    cp->lc = lc;
    std::vector<tt_tis> vd = {tp, tq, tr, ts};
    std::vector<uint8_t> vnz, wnz;
    chol_maps(X, vd, vnz, wnz);
    TT_TRY(new_meta_tensor(ctx, vd, vnz, &cp->Vmeta));
    TT_TRY(new_meta_tensor(ctx, vd, wnz, &cp->Wmeta));
    // Bh: B's blocks with r_t <= s_t (the antisymmetric Bm's independent half), and its strict view
    const size_t rp = b.find(r), sp_ = b.find(s);
    std::vector<uint8_t> hnz(B->nblocks, 0), snz(B->nblocks, 0);
    std::vector<int> id(B->order), sw(B->order);
    for (int d = 0; d < B->order; ++d) id[d] = sw[d] = d;
    sw[rp] = (int)sp_;
    sw[sp_] = (int)rp;
    int32_t bc[TT_MAX_ORDER], bsc[TT_MAX_ORDER];
    std::vector<int64_t> swap_of(B->nblocks, -1);
    for (int64_t x = 0; x < B->nblocks; ++x) {
      B->block_coords(x, bc);
      for (int d = 0; d < B->order; ++d) bsc[sw[d]] = bc[d];
      swap_of[x] = B->block_id(bsc);
      const bool nzm = B->nz[x] || B->nz[swap_of[x]];       // Bm(x) = B(x) - B(swap x)^T
      hnz[x] = (nzm && bc[rp] <= bc[sp_]) ? 1 : 0;
      snz[x] = (hnz[x] && bc[rp] < bc[sp_]) ? 1 : 0;
    }
    TT_TRY(new_meta_tensor(ctx, B->dims, hnz, &cp->Bh));
    TT_TRY(new_meta_tensor(ctx, B->dims, snz, &cp->Bs));
    for (int64_t x = 0; x < B->nblocks; ++x) {     // Bs shares Bh's storage
      cp->Bs->blk_off[x] = cp->Bs->gblk_off[x] = snz[x] ? cp->Bh->blk_off[x] : -1;
      if (snz[x]) cp->Bs->owner[x] = TT_REPLICATED;
    }
    cp->Bs->packed_elems = cp->Bs->storage_elems = cp->Bh->packed_elems;
    // formation owner of each Bh block: the rank holding both B(x) and B(swap x) whole (replicated
    // blocks are held everywhere); B pairs split across ranks -> all-gather B instead
    cp->colocated = true;
    std::vector<uint8_t> mine(B->nblocks, 0);
    for (int64_t x = 0; x < B->nblocks; ++x) {
      if (!hnz[x]) continue;
      const int64_t y = swap_of[x];
      int32_t ox = B->nz[x] ? B->owner[x] : TT_REPLICATED, oy = B->nz[y] ? B->owner[y] : TT_REPLICATED;
      if ((B->nz[x] && !B->parts[x].empty()) || (B->nz[y] && !B->parts[y].empty()) || ox == TT_SPLIT || oy == TT_SPLIT) {
        cp->colocated = false;
        break;
      }
      const int32_t f = (ox == TT_REPLICATED) ? oy : ox;
      if (oy != TT_REPLICATED && oy != f) { cp->colocated = false; break; }
      cp->Bh->owner[x] = f;
      mine[x] = (f == TT_REPLICATED || f == ctx->rank) ? 1 : 0;
    }
    Needs need(ctx->nranks);
    if (cp->colocated) {
      for (int rr = 0; rr < ctx->nranks; ++rr)
        for (int64_t x = 0; x < B->nblocks; ++x)
          if (hnz[x]) need[rr].push_back({0, x, 0, cp->Bh->block_volume(x)});
      TT_TRY(build_gather(ctx, need, {cp->Bh}, cp->hgather));
    } else {
      for (int64_t x = 0; x < B->nblocks; ++x) {
        if (hnz[x]) cp->Bh->owner[x] = TT_REPLICATED;
        mine[x] = hnz[x];
      }
      for (int rr = 0; rr < ctx->nranks; ++rr)
        for (int64_t x = 0; x < B->nblocks; ++x)
          if (B->nz[x]) need[rr].push_back({0, x, 0, B->block_volume(x)});
      TT_TRY(build_gather(ctx, need, {B}, cp->bgather));
    }
    // Bh = B - B(r<->s) on this rank's Bh blocks
    TT_TRY(local_add_plan(ctx, cp->Bh, B, id, 0.0, cp->copy_plan, &mine));
    TT_TRY(local_add_plan(ctx, cp->Bh, B, sw, 1.0, cp->swap_plan, &mine));
    // SPMD plans for this rank's C parts: V map (algorithmic FLOPs) and W map (executed pairs)
    ContractOpts g;
    g.no_gather = true;
    g.tag = "|cholV";
    bool dummy;
    TT_TRY(get_contract_plan(ctx, C, cl, cp->Vmeta, vl, B, bl, beta, cp->vplan, &dummy, g));
    g.tag = "|cholW";
    TT_TRY(get_contract_plan(ctx, C, cl, cp->Wmeta, vl, B, bl, beta, cp->wplan, &dummy, g));
    const ContractPlan& gp = *cp->wplan;
    // units: my C parts grouped by the (p,q) tile coordinates; W rows restricted when C's dim 0 is p
    const bool rows_on_p = c[0] == p;
    const int cp_pos = (int)c.find(p), cq_pos = (int)c.find(q);
    struct Unit {
      int32_t tp, tq;
      std::vector<std::pair<int64_t, int64_t>> wrows;
      std::vector<PartSel> cparts;
    };
    std::map<std::pair<int32_t, int32_t>, Unit> units;
    int32_t cc[TT_MAX_ORDER];
    for (const auto& mp : gp.my) {
      const int64_t cb = gp.ht.cblk[mp.g];
      C->block_coords(cb, cc);
      Unit& u = units[{cc[cp_pos], cc[cq_pos]}];
      u.tp = cc[cp_pos];
      u.tq = cc[cq_pos];
      u.cparts.push_back({cb, mp.lo, mp.hi});
      if (rows_on_p) u.wrows.push_back({mp.lo, mp.hi});
      else u.wrows.push_back({0, tp->size(u.tp)});
    }
    auto row_blocks = [&](const Unit& u, std::vector<int64_t>& out) {
      out.clear();
      for (int32_t a2 = 0; a2 < tr->ntiles(); ++a2)
        for (int32_t b2 = 0; b2 < ts->ntiles(); ++b2) {
          const int64_t vb = (((int64_t)u.tp * tq->ntiles() + u.tq) * tr->ntiles() + a2) * ts->ntiles() + b2;
          if (wnz[vb]) out.push_back(vb);
        }
    };
    // workspace: Bh then the W batches; without room for Bh plus the largest W row, two passes
    std::vector<int64_t> rb;
    int64_t max_uel = 0;
    for (auto& kv : units) {
      row_blocks(kv.second, rb);
      int64_t uel = 0;
      for (int64_t vb : rb) uel += (cp->Wmeta->block_volume(vb) + 1) / 2 * 2;
      max_uel = std::max(max_uel, uel);
    }
    if (const char* f2 = getenv("TT_CHOL_TWO_PASS")) cp->two_pass = atoi(f2) != 0;
    const int64_t bh_elems = (cp->Bh->packed_elems + 31) / 32 * 32;
    if (ws_elems < bh_elems + max_uel) cp->two_pass = true;
    if (cp->two_pass) {    // B is read directly: all-gather it (not Bh)
      cp->hgather = GatherPlan();
      if (cp->colocated) {
        Needs nb(ctx->nranks);
        for (int rr = 0; rr < ctx->nranks; ++rr)
          for (int64_t x = 0; x < B->nblocks; ++x)
            if (B->nz[x]) nb[rr].push_back({0, x, 0, B->block_volume(x)});
        TT_TRY(build_gather(ctx, nb, {B}, cp->bgather));
      }
    }
    if (ws_elems < max_uel)
      return fail(TT_E_OOM, "workspace holds %lld doubles; one (p,q) row of W needs %lld", (long long)ws_elems,
                  (long long)max_uel);
    const int64_t w_off = cp->two_pass ? 0 : bh_elems;
    double* wbase = (double*)workspace + w_off;
    const int64_t w_elems = ws_elems - w_off;
    if (!cp->two_pass) {
      cp->Bh->data = cp->Bs->data = (double*)workspace;
      cp->Bh->capacity = cp->Bs->capacity = bh_elems;
    }
    auto flush = [&](std::vector<const Unit*>& cur) -> tt_status {
      if (cur.empty()) return TT_OK;
      CholBatch bt;
      std::vector<uint8_t> bnz(wnz.size(), 0);
      std::vector<int64_t> rb;
      for (const Unit* u : cur) {
        auto rows = u->wrows;
        std::sort(rows.begin(), rows.end());
        std::vector<std::pair<int64_t, int64_t>> mr;
        for (auto& x : rows) {
          if (!mr.empty() && x.first <= mr.back().second) mr.back().second = std::max(mr.back().second, x.second);
          else mr.push_back(x);
        }
        row_blocks(*u, rb);
        for (int64_t vb : rb) {
          bnz[vb] = 1;
          for (auto& x : mr) bt.wopt.sel.push_back({vb, x.first, x.second});
        }
        for (const PartSel& ps : u->cparts) bt.copt.sel.push_back(ps);
      }
      TT_TRY(new_meta_tensor(ctx, vd, bnz, &bt.Wb));
      if (bt.Wb->packed_elems > w_elems) {
        const long long need = (long long)bt.Wb->packed_elems;
        delete bt.Wb;
        return fail(TT_E_OOM, "workspace after Bh holds %lld doubles; one (p,q) row of W needs %lld",
                    (long long)w_elems, need);
      }
      bt.Wb->data = wbase;
      bt.Wb->capacity = w_elems;
      bt.wopt.local = bt.copt.local = true;
      const size_t bi = cp->batches.size();
      bt.wopt.tag = "|cholWb" + std::to_string(bi);
      bt.copt.tag = "|cholCb" + std::to_string(bi);
      cp->batches.push_back(bt);
      cur.clear();
      return TT_OK;
    };
    std::vector<const Unit*> cur;
    int64_t cur_elems = 0;
    for (auto& kv : units) {
      const Unit& u = kv.second;
      row_blocks(u, rb);
      int64_t uel = 0;
      for (int64_t vb : rb) uel += (cp->Wmeta->block_volume(vb) + 1) / 2 * 2;
      if (!cur.empty() && cur_elems + uel > w_elems) {
        TT_TRY(flush(cur));
        cur_elems = 0;
      }
      cur.push_back(&u);
      cur_elems += uel;
    }
    TT_TRY(flush(cur));
    plan_put(ctx, keybuf, cp);
  }
  const std::string L = cp->lc;
  const std::string x1 = std::string(1, p) + r + L, x2 = std::string(1, q) + s + L;   // W = X(prL) X(qsL)
  std::string bsw(bl);                                                              // B with r <-> s
  std::swap(bsw[b.find(r)], bsw[b.find(s)]);
  const std::string vsw = std::string(1, p) + q + s + r;                              // W read as (p,q,s,r)
  if (ctx->prepare_only) {   // build every batch plan now (they are cached), launch nothing
    for (auto& bt : cp->batches) {
      std::shared_ptr<ContractPlan> pw, pu, px;
      bool dummy;
      TT_TRY(get_contract_plan(ctx, bt.Wb, vl, X, x1.c_str(), X, x2.c_str(), 0.0, pw, &dummy, bt.wopt));
      if (cp->two_pass) {
        TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vl, B, bl, beta, pu, &dummy, bt.copt));
        TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vl, B, bsw.c_str(), 1.0, px, &dummy, bt.copt));
      } else {
        TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vl, cp->Bh, bl, beta, pu, &dummy, bt.copt));
        TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vsw.c_str(), cp->Bs, bl, 1.0, px, &dummy, bt.copt));
      }
    }
    return TT_OK;
  }
  reset_stats(ctx);
  trace("cholesky: plans ready, batches", (long long)cp->batches.size());
  TT_TRY(run_gather(ctx, cp->bgather, {B}));
  trace("B gathered, runs", (long long)(cp->bgather.recv.size() + cp->bgather.send.size()));
  if (!cp->two_pass) {
    TT_TRY(run_local_add(ctx, *cp->copy_plan, cp->Bh, B, 0.0, 1.0));
    TT_TRY(run_local_add(ctx, *cp->swap_plan, cp->Bh, B, 1.0, -1.0));
    trace("Bh formed");
    TT_TRY(run_gather(ctx, cp->hgather, {cp->Bh}));
    trace("Bh gathered, runs", (long long)(cp->hgather.recv.size() + cp->hgather.send.size()));
  }
  double exec = 0, build = 0;
  int64_t tasks = 0;
  for (auto& bt : cp->batches) {
    std::shared_ptr<ContractPlan> pw, pu, px;
    bool dummy;
    TT_TRY(get_contract_plan(ctx, bt.Wb, vl, X, x1.c_str(), X, x2.c_str(), 0.0, pw, &dummy, bt.wopt));
    TT_TRY(launch_plan(ctx, *pw, bt.Wb, vl, 0.0, 1.0, X, x1.c_str(), X, x2.c_str()));
    build += pw->flops;
    if (cp->two_pass) {
      TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vl, B, bl, beta, pu, &dummy, bt.copt));
      TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vl, B, bsw.c_str(), 1.0, px, &dummy, bt.copt));
      TT_TRY(launch_plan(ctx, *pu, C, cl, beta, alpha, bt.Wb, vl, B, bl));
      TT_TRY(launch_plan(ctx, *px, C, cl, 1.0, -alpha, bt.Wb, vl, B, bsw.c_str()));
      exec += pu->flops + px->flops;
      tasks += pu->tasks + px->tasks;
    } else {
      TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vl, cp->Bh, bl, beta, pu, &dummy, bt.copt));
      TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vsw.c_str(), cp->Bs, bl, 1.0, px, &dummy, bt.copt));
      TT_TRY(launch_plan(ctx, *pu, C, cl, beta, alpha, bt.Wb, vl, cp->Bh, bl));
      TT_TRY(launch_plan(ctx, *px, C, cl, 1.0, -alpha, bt.Wb, vsw.c_str(), cp->Bs, bl));
      exec += pu->flops + px->flops;
      tasks += pu->tasks + px->tasks;
    }
    if (trace.on && (&bt - &cp->batches[0]) % 16 == 0) trace("batch done", (long long)(&bt - &cp->batches[0]));
  }
  trace("cholesky done");
  ctx->last.c_blocks = (int64_t)cp->wplan->my.size();
  ctx->last.tasks = tasks;
  ctx->last.flops = cp->vplan->flops;       // algorithmic: the defined contraction over V's block map
  ctx->last.aux_flops = build + exec;       // executed: W build + consume (passes 1 and 2, or two-pass)
  ctx->last.gathered_bytes = cp->bgather.recv_bytes + (cp->two_pass ? 0 : cp->hgather.recv_bytes);
  ctx->last.work_items = (int64_t)cp->batches.size();
  return TT_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// three-operand contraction evaluated through an intermediate (PAPER Eqs.
// cc9-cc11, P293-311: the n_o^4 n_u^4 term 1/4 v^{ef}_{mn} t^{ij}_{ef} t^{mn}_{ab} becomes
// I^{ij}_{mn} = v^{ef}_{mn} t^{ij}_{ef} followed by 1/4 I^{ij}_{mn} t^{mn}_{ab}, "total numerical cost
// proportional to n_o^4 n_u^2").  Every pairing is costed on the block maps (reading R26) and the
// cheapest is executed as two binary contractions of the DMMA path.

namespace {

struct C3Plan {
  tt_tensor I = nullptr;
  std::string i_lbl, x_lbl, y_lbl, z_lbl;
  int pair = 0;
  tt_tensor X = nullptr, Y = nullptr, Z = nullptr;
  double flops[3] = {0, 0, 0}, naive = 0;
  ~C3Plan() { delete I; }
};

struct C3Cand {
  std::string il;
  std::vector<tt_tis> idims;
  std::vector<uint8_t> inz;
  double flops1 = 0, flops2 = 0;
};

// intermediate of the pair (X, Y) when the third operand is Z: the labels of X then Y that survive
// (appear in Z or in C), on their tiled spaces; its block map = the blocks that receive a task.
tt_status c3_candidate(tt_ctx ctx, tt_tensor C, const std::string& cl, tt_tensor X, const std::string& xl,
                       tt_tensor Y, const std::string& yl, tt_tensor Z, const std::string& zl, C3Cand& cd) {
  cd.il.clear();
  cd.idims.clear();
  for (int s = 0; s < 2; ++s) {
    const std::string& l = s ? yl : xl;
    tt_tensor T = s ? Y : X;
    for (size_t d = 0; d < l.size(); ++d) {
      const char x = l[d];
      const bool keep = zl.find(x) != std::string::npos || cl.find(x) != std::string::npos;
      if (keep && cd.il.find(x) == std::string::npos) {
        cd.il.push_back(x);
        cd.idims.push_back(T->dims[d]);
      }
    }
  }
  if (cd.il.empty() || cd.il.size() > (size_t)TT_MAX_ORDER)
    return fail(TT_E_UNSUPPORTED, "intermediate of order %zu", cd.il.size());
  tt_tensor Id;
  int64_t nb = 1;
  for (auto d : cd.idims) nb *= d->ntiles();
  TT_TRY(new_meta_tensor(ctx, cd.idims, std::vector<uint8_t>(nb, 1), &Id));
  std::unique_ptr<tt_tensor_s> hold(Id);
  Analysis a1;
  TT_TRY(analyse(Id, cd.il.c_str(), X, xl.c_str(), Y, yl.c_str(), a1));
  HostTasks h1;
  enumerate_tasks(a1, Id, X, Y, h1);
  cd.inz.assign(nb, 0);
  cd.flops1 = 0;
  for (size_t g = 0; g < h1.cblk.size(); ++g)
    if (h1.ptr[g + 1] > h1.ptr[g]) {
      cd.inz[h1.cblk[g]] = 1;
      cd.flops1 += (double)h1.cost[g];
    }
  Id->nz = cd.inz;
  tensor_finish(Id);
  Analysis a2;
  TT_TRY(analyse(C, cl.c_str(), Id, cd.il.c_str(), Z, zl.c_str(), a2));
  HostTasks h2;
  enumerate_tasks(a2, C, Id, Z, h2);
  cd.flops2 = 0;
  for (int64_t c : h2.cost) cd.flops2 += (double)c;
  return TT_OK;
}

// multiply-adds of the unfactorized loop: one product A*B*D per combination of all label values whose
// four blocks (C, A, B, D) are non-zero; -1 when the label tile grid is too large to enumerate
double c3_naive_macs(tt_tensor C, const std::string& cl, tt_tensor const T[3], const std::string L[3]) {
  std::string uni = cl;
  std::vector<tt_tis> lt;
  for (size_t d = 0; d < cl.size(); ++d) lt.push_back(C->dims[d]);
  for (int s = 0; s < 3; ++s)
    for (size_t d = 0; d < L[s].size(); ++d)
      if (uni.find(L[s][d]) == std::string::npos) { uni.push_back(L[s][d]); lt.push_back(T[s]->dims[d]); }
  double ntup = 1;
  for (auto t : lt) ntup *= t->ntiles();
  if (ntup > 5e7) return -1;
  const int nu = (int)uni.size();
  std::vector<int32_t> tile(nu, 0);
  double macs = 0;
  for (int64_t k = 0; k < (int64_t)ntup; ++k) {
    int64_t r = k;
    for (int u = nu - 1; u >= 0; --u) { tile[u] = (int32_t)(r % lt[u]->ntiles()); r /= lt[u]->ntiles(); }
    auto nzof = [&](tt_tensor T, const std::string& l) {
      int64_t b = 0;
      for (size_t d = 0; d < l.size(); ++d) b = b * T->grid[d] + tile[uni.find(l[d])];
      return T->nz[b] != 0;
    };
    if (!nzof(C, cl) || !nzof(T[0], L[0]) || !nzof(T[1], L[1]) || !nzof(T[2], L[2])) continue;
    double v = 1;
    for (int u = 0; u < nu; ++u) v *= (double)lt[u]->size(tile[u]);
    macs += v;
  }
  return macs;
}

}  // namespace

extern "C" {

tt_status tt_contract3(tt_ctx ctx, tt_tensor C, const char* cl, double beta, double alpha, tt_tensor A,
                       const char* al, tt_tensor B, const char* bl, tt_tensor D, const char* dl, void* workspace,
                       int64_t ws_elems, tt_contract3_info* info) {
  NvtxRange nvtx_("tt_contract3");
  if (!ctx || !C || !A || !B || !D || !cl || !al || !bl || !dl) return fail(TT_E_ARG, "NULL argument");
  TT_TRY(check_labels(cl, C, "C"));
  TT_TRY(check_labels(al, A, "A"));
  TT_TRY(check_labels(bl, B, "B"));
  TT_TRY(check_labels(dl, D, "D"));
  const std::string L[4] = {cl, al, bl, dl};
  // every label in exactly two of the four operands (no batch / dangling labels, S380)
  for (int s = 0; s < 4; ++s)
    for (char x : L[s]) {
      int n = 0;
      for (int q = 0; q < 4; ++q) n += L[q].find(x) != std::string::npos;
      if (n != 2) return fail(TT_E_LABEL, "label '%c' appears in %d of C, A, B, D (must be exactly 2)", x, n);
    }
  char keybuf[600];
  snprintf(keybuf, sizeof(keybuf), "c3|%llu.%llu|%llu.%llu|%llu.%llu|%llu.%llu|%s|%s|%s|%s",
           (unsigned long long)C->uid, (unsigned long long)C->version, (unsigned long long)A->uid,
           (unsigned long long)A->version, (unsigned long long)B->uid, (unsigned long long)B->version,
           (unsigned long long)D->uid, (unsigned long long)D->version, cl, al, bl, dl);
  auto cp = cached<C3Plan>(ctx, keybuf);
  double cand_flops[3] = {0, 0, 0};
  double naive = 0;
  if (!cp) {
    cp = std::make_shared<C3Plan>();
    tt_tensor T[3] = {A, B, D};
    const std::string TL[3] = {al, bl, dl};
    static const int pairs[3][3] = {{0, 1, 2}, {0, 2, 1}, {1, 2, 0}};   // (X, Y, Z): (AB)D, (AD)B, (BD)A
    C3Cand best;
    int bi = -1;
    for (int p = 0; p < 3; ++p) {
      const int x = pairs[p][0], y = pairs[p][1], z = pairs[p][2];
      C3Cand cd;
      tt_status st = c3_candidate(ctx, C, cl, T[x], TL[x], T[y], TL[y], T[z], TL[z], cd);
      if (st == TT_E_UNSUPPORTED) { cand_flops[p] = -1; continue; }
      TT_TRY(st);
      cand_flops[p] = cd.flops1 + cd.flops2;
      if (bi < 0 || cand_flops[p] < cand_flops[bi]) { bi = p; best = cd; }
    }
    if (bi < 0) return fail(TT_E_UNSUPPORTED, "no pairing has a supported intermediate");
    naive = c3_naive_macs(C, cl, T, TL);
    cp->pair = bi;
    cp->X = T[pairs[bi][0]]; cp->x_lbl = TL[pairs[bi][0]];
    cp->Y = T[pairs[bi][1]]; cp->y_lbl = TL[pairs[bi][1]];
    cp->Z = T[pairs[bi][2]]; cp->z_lbl = TL[pairs[bi][2]];
    cp->i_lbl = best.il;
    TT_TRY(new_meta_tensor(ctx, best.idims, best.inz, &cp->I));
    cp->I->ctx = ctx;
    // remember the costs with the plan (returned on every call)
    cp->flops[0] = cand_flops[0]; cp->flops[1] = cand_flops[1]; cp->flops[2] = cand_flops[2];
    cp->naive = naive;
    plan_put(ctx, keybuf, cp);
  }
  const int64_t need = (cp->I->storage_elems + 1) / 2 * 2;
  if (info) {
    info->pair = cp->pair;
    memset(info->i_lbl, 0, sizeof(info->i_lbl));
    memcpy(info->i_lbl, cp->i_lbl.data(), cp->i_lbl.size());
    for (int p = 0; p < 3; ++p) info->flops[p] = cp->flops[p];
    info->naive_macs = cp->naive;
    info->ws_elems = need;
  }
  if (!workspace) return TT_OK;   // query: pairing, costs and workspace size only
  if (ws_elems < need) return fail(TT_E_ARG, "workspace holds %lld doubles, the intermediate needs %lld",
                                   (long long)ws_elems, (long long)need);
  TT_TRY(tt_tensor_bind(cp->I, workspace, ws_elems));
  TT_TRY(tt_contract(ctx, cp->I, cp->i_lbl.c_str(), 0.0, 1.0, cp->X, cp->x_lbl.c_str(), cp->Y, cp->y_lbl.c_str()));
  const tt_stats first = ctx->last;
  TT_TRY(tt_contract(ctx, C, cl, beta, alpha, cp->I, cp->i_lbl.c_str(), cp->Z, cp->z_lbl.c_str()));
  ctx->last.flops += first.flops;
  ctx->last.tasks += first.tasks;
  ctx->last.gathered_bytes += first.gathered_bytes;
  ctx->last.bytes += first.bytes;
  return TT_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// perturbative triples correction (T), PAPER Eqs. cc14, tensort, abt, tensort2
// (P343-413).  The inputs are copied into dense, permuted layouts in the workspace (re-tiling kernel),
// then one fused kernel launch per batch of units (occupied triple i<j<k x virtual box triple) forms W in
// shared memory through three GEMMs (tt_triples.cu) and reduces (W + V1) W / D (reading R28) into one
// partial per unit; a fixed-order final sum (R12) and, with nranks > 1, an NCCL all-reduce give E(T).
// Units are enumerated box-major (consecutive CTAs share the virtual slices in L2) and split into
// contiguous equal ranges over the ranks; spin-forbidden units (sum of box spins != sum of occupied spins)
// are skipped -- W vanishes there for the spin maps of reading R7.

namespace {

struct RetileOp {
  DevMem mem;                // workspace regions of the device arrays below
  tt_tensor dst = nullptr;   // meta tensor on the dense tiling, storage in the workspace
  tt_tensor src = nullptr;
  std::vector<int32_t> sdim;
  RetileBlk* d_blks = nullptr;
  Segment* d_segs = nullptr;
  int64_t nseg = 0, ws_pos = 0;
  int32_t* d_g2t[TT_MAX_ORDER] = {};
};

struct TripPlan {
  DevMem mem;                                 // workspace regions of the device arrays below
  tt_tis fullO = nullptr, fullV = nullptr;   // one tile over the whole space (dense copies)
  RetileOp rt[5];                             // VO (O,O,O,V), VV (V,O,V,V), T2 (O,O,V,V), VD (O,O,V,V), T1 (V,O)
  int2* d_units = nullptr;
  int2* d_pairs = nullptr;                    // pair variant: (first unit, count) per CTA
  int64_t npairs = 0;
  int4* d_box3 = nullptr;
  int4* d_trip = nullptr;
  int32_t* d_box_lo = nullptr;
  int32_t* d_box_ext = nullptr;
  double* d_partials = nullptr;
  int64_t unit0 = 0, nunits = 0, nunits_total = 0;
  int32_t o_half = 0, v_half = 0;
  int64_t ws_need = 0;
  int64_t blk_pos[4] = {0, 0, 0, 0}, blk_n[4] = {0, 0, 0, 0};   // blocked copies (QT2, QVV, PVO, PT2)
  int32_t nbox = 0;
  int32_t kpo = 0, kpv = 0, ko2 = 0, kv2 = 0;   // padded summed rows of the blocked copies
  tt_triples_info info{};
  ~TripPlan() {
    for (auto& r : rt) delete r.dst;
    delete fullO;
    delete fullV;
  }
};

tt_tis full_tiling(tt_tis t) {
  tt_tis r = new tt_tis_s();
  r->is = t->is;
  r->uid = g_uid++;
  r->offsets = {0, t->offsets.back()};
  r->spin = {0};
  return r;
}

int64_t ordered_count3(int64_t lo0, int64_t n0, int64_t lo1, int64_t n1, int64_t lo2, int64_t n2) {
  // x<y<z with x in [lo0, lo0+n0), y in [lo1, ...), z in [lo2, ...), ranges ordered and equal or disjoint
  const bool e01 = lo0 == lo1, e12 = lo1 == lo2;
  if (e01 && e12) return n0 * (n0 - 1) * (n0 - 2) / 6;
  if (e01) return n0 * (n0 - 1) / 2 * n2;
  if (e12) return n0 * n1 * (n1 - 1) / 2;
  return n0 * n1 * n2;
}

tt_status build_retile(tt_ctx ctx, RetileOp& op) {
  tt_tensor D = op.dst, Sx = op.src;
  TT_TRY(ensure_dev(Sx));
  std::vector<RetileBlk> blks;
  std::vector<Segment> segs;
  int32_t c[TT_MAX_ORDER];
  for (int64_t b = 0; b < D->nblocks; ++b) {
    if (!D->nz[b]) continue;
    D->block_coords(b, c);
    RetileBlk rb{};
    rb.dst_off = D->blk_off[b];
    for (int q = 0; q < D->order; ++q) {
      rb.org[q] = (int32_t)D->dims[q]->offsets[c[q]];
      rb.ext[q] = (int32_t)D->dims[q]->size(c[q]);
    }
    const int64_t vol = D->block_volume(b);
    for (int64_t e = 0; e < vol; e += 32768)
      segs.push_back({(int32_t)blks.size(), 0, e, std::min(vol, e + 32768)});
    blks.push_back(rb);
  }
  TT_TRY(dev_alloc(ctx, op.mem, &op.d_blks, std::max<size_t>(1, blks.size())));
  TT_TRY(dev_alloc(ctx, op.mem, &op.d_segs, std::max<size_t>(1, segs.size())));
  if (!blks.empty()) TT_CUDA(cudaMemcpy(op.d_blks, blks.data(), blks.size() * sizeof(RetileBlk), cudaMemcpyHostToDevice));
  if (!segs.empty()) TT_CUDA(cudaMemcpy(op.d_segs, segs.data(), segs.size() * sizeof(Segment), cudaMemcpyHostToDevice));
  op.nseg = (int64_t)segs.size();
  for (int q = 0; q < Sx->order; ++q) {
    tt_tis t = Sx->dims[q];
    std::vector<int32_t> g2t(t->offsets.back());
    for (int x = 0; x < t->ntiles(); ++x)
      for (int64_t g = t->offsets[x]; g < t->offsets[x + 1]; ++g) g2t[g] = x;
    TT_TRY(dev_alloc(ctx, op.mem, &op.d_g2t[q], g2t.size()));
    TT_CUDA(cudaMemcpy(op.d_g2t[q], g2t.data(), g2t.size() * 4, cudaMemcpyHostToDevice));
  }
  return TT_OK;
}

tt_status run_retile(tt_ctx ctx, const RetileOp& op) {
  RetileParams p{};
  p.order = op.src->order;
  p.src = op.src->data;
  p.dst = op.dst->data;
  p.blks = op.d_blks;
  p.segs = op.d_segs;
  for (int q = 0; q < p.order; ++q) {
    p.g2t[q] = op.d_g2t[q];
    p.toff[q] = op.src->d_toff[q];
    p.sgrid[q] = op.src->grid[q];
    p.sdim[q] = op.sdim[q];
  }
  p.sblk_off = op.src->d_blk_off;
  Launch L(ctx, "tt_retile");
  TT_CUDA(launch_retile(p, op.nseg, ctx->stream));
  return TT_OK;
}

}  // namespace

extern "C" {

tt_status tt_triples_energy(tt_ctx ctx, tt_tensor T1, tt_tensor T2, tt_tensor Vooov, tt_tensor Vvovv,
                            tt_tensor Voovv, const double* eps_o, const double* eps_v, void* workspace,
                            int64_t ws_elems, double* energy, tt_triples_info* info) {
  NvtxRange nvtx_("tt_triples_energy");
  if (!ctx || !T1 || !T2 || !Vooov || !Vvovv || !Voovv) return fail(TT_E_ARG, "NULL argument");
  if (T1->order != 2 || T2->order != 4 || Vooov->order != 4 || Vvovv->order != 4 || Voovv->order != 4)
    return fail(TT_E_ARG, "T1 (a,i) order 2; T2 (a,b,i,j), Vooov (i,j,m,a), Vvovv (e,i,a,b), Voovv (i,j,a,b) order 4");
  tt_tis tV = T1->dims[0], tO = T1->dims[1];
  const tt_tis want[5][4] = {{tV, tO, nullptr, nullptr}, {tV, tV, tO, tO}, {tO, tO, tO, tV}, {tV, tO, tV, tV}, {tO, tO, tV, tV}};
  const tt_tensor ins[5] = {T1, T2, Vooov, Vvovv, Voovv};
  const char* names[5] = {"T1", "T2", "Vooov", "Vvovv", "Voovv"};
  for (int x = 1; x < 5; ++x)
    for (int d = 0; d < 4; ++d)
      if (ins[x]->dims[d] != want[x][d])
        return fail(TT_E_TILING, "%s dim %d: must be T1's %s tiled index space object (S413)", names[x], d,
                    want[x][d] == tO ? "occupied" : "virtual");
  for (int x = 0; x < 5; ++x) {
    if (ins[x]->compact || ins[x]->any_split || ins[x]->view_of)
      return fail(TT_E_UNSUPPORTED, "%s: compact, row-split or view inputs", names[x]);
    // the kernel prunes units and m / e ranges by the spins of the index ranges (R28, R6/R7): valid
    // only if every non-zero input block obeys the spin rule (upper dims {0,1} | lower {2,3}; T1 {0}|{1})
    int32_t c[TT_MAX_ORDER];
    for (int64_t b = 0; b < ins[x]->nblocks; ++b) {
      if (!ins[x]->nz[b]) continue;
      ins[x]->block_coords(b, c);
      int su = 0, sl = 0;
      for (int d = 0; d < ins[x]->order; ++d) {
        const int s = ins[x]->dims[d]->spin[c[d]];
        if (d < ins[x]->order / 2) su += s;
        else sl += s;
      }
      if (su != sl)
        return fail(TT_E_UNSUPPORTED, "%s: non-zero block %lld breaks the spin rule the (T) kernel prunes by "
                    "(use the spin block maps of reading R7 on alpha/beta spaces)", names[x], (long long)b);
    }
    if (ctx->nranks > 1)
      for (int64_t b = 0; b < ins[x]->nblocks; ++b)
        if (ins[x]->nz[b] && ins[x]->owner[b] != TT_REPLICATED)
          return fail(TT_E_UNSUPPORTED, "%s: with nranks > 1 every input block must be TT_REPLICATED", names[x]);
  }
  const int64_t nO = tO->offsets.back(), nV = tV->offsets.back();
  if (nO < 3 || nV < 3) return fail(TT_E_ARG, "need at least 3 occupied and 3 virtual indices");
  for (size_t q = 0; q < tV->is->rb.size(); ++q)
    if ((tV->is->re[q] - tV->is->rb[q]) % 2)
      return fail(TT_E_UNSUPPORTED, "virtual ranges must have even sizes (16-byte staging of the fused kernel)");
  char keybuf[400];
  snprintf(keybuf, sizeof(keybuf), "trip|%llu.%llu|%llu.%llu|%llu.%llu|%llu.%llu|%llu.%llu",
           (unsigned long long)T1->uid, (unsigned long long)T1->version, (unsigned long long)T2->uid,
           (unsigned long long)T2->version, (unsigned long long)Vooov->uid, (unsigned long long)Vooov->version,
           (unsigned long long)Vvovv->uid, (unsigned long long)Vvovv->version, (unsigned long long)Voovv->uid,
           (unsigned long long)Voovv->version);
  auto tp = cached<TripPlan>(ctx, keybuf);
  if (!tp) {
    tp = std::make_shared<TripPlan>();
    tp->fullO = full_tiling(tO);
    tp->fullV = full_tiling(tV);
    tt_tis fO = tp->fullO, fV = tp->fullV;
    // dense copies: dims (dst order) and, per source dim, the dst dim holding it
    struct Spec { tt_tensor src; std::vector<tt_tis> dims; std::vector<int32_t> sdim; };
    const Spec specs[5] = {{Vooov, {fO, fO, fO, fV}, {0, 1, 2, 3}},
                           {Vvovv, {fV, fO, fV, fV}, {0, 1, 2, 3}},
                           {T2, {fO, fO, fV, fV}, {2, 3, 0, 1}},       // t^{ij}_{ab}: (a,b,i,j) -> (i,j,a,b)
                           {Voovv, {fO, fO, fV, fV}, {0, 1, 2, 3}},
                           {T1, {fV, fO}, {0, 1}}};
    int64_t base = 0;
    for (int x = 0; x < 5; ++x) {
      TT_TRY(new_meta_tensor(ctx, specs[x].dims, std::vector<uint8_t>(1, 1), &tp->rt[x].dst));
      tp->rt[x].src = specs[x].src;
      tp->rt[x].sdim = specs[x].sdim;
      tp->rt[x].ws_pos = base;
      base += (tp->rt[x].dst->packed_elems + 31) / 32 * 32;
    }
    // virtual boxes: each range of V cut into boxes of kTripBox (never straddle spin, S39)
    std::vector<int32_t> box_lo, box_ext;
    std::vector<int8_t> box_spin;
    for (size_t q = 0; q < tV->is->rb.size(); ++q)
      for (int64_t x = tV->is->rb[q]; x < tV->is->re[q]; x += kTripBox) {
        box_lo.push_back((int32_t)x);
        box_ext.push_back((int32_t)std::min<int64_t>(kTripBox, tV->is->re[q] - x));
        box_spin.push_back(tV->is->rspin[q]);
      }
    const int nb = (int)box_lo.size();
    tp->nbox = nb;
    std::vector<int4> box3;
    std::vector<int64_t> box3_n;
    for (int a = 0; a < nb; ++a) for (int b = a; b < nb; ++b) for (int c = b; c < nb; ++c) {
      const int64_t n = ordered_count3(box_lo[a], box_ext[a], box_lo[b], box_ext[b], box_lo[c], box_ext[c]);
      if (n > 0) { box3.push_back({a, b, c, box_spin[a] + box_spin[b] + box_spin[c]}); box3_n.push_back(n); }
    }
    // occupied triples i<j<k with their spin sums (spin of the range holding the index)
    std::vector<int8_t> ospin(nO, 0);
    for (size_t q = 0; q < tO->is->rb.size(); ++q)
      for (int64_t x = tO->is->rb[q]; x < tO->is->re[q]; ++x) ospin[x] = tO->is->rspin[q];
    std::vector<int4> trip;
    for (int i = 0; i < nO; ++i) for (int j = i + 1; j < nO; ++j) for (int k = j + 1; k < nO; ++k)
      trip.push_back({i, j, k, ospin[i] + ospin[j] + ospin[k]});
    std::vector<int2> units;
    double alg = 0;
    const double per = 18.0 * (double)(nO + nV);
    for (size_t b3 = 0; b3 < box3.size(); ++b3)
      for (size_t t = 0; t < trip.size(); ++t)
        if (box3[b3].w == trip[t].w) { units.push_back({(int)b3, (int)t}); }
    const int64_t U = (int64_t)units.size();
    if (U >= (1ll << 31)) return fail(TT_E_UNSUPPORTED, "%lld (T) units exceed the int32 unit index", (long long)U);
    tp->nunits_total = U;
    // spin split points (R6: alpha = the first range) when each space is exactly (alpha, beta)
    auto half = [](tt_tis t) -> int32_t {
      const tt_is s = t->is;
      return (s->rb.size() == 2 && s->rspin[0] == 1 && s->rspin[1] == -1) ? (int32_t)s->re[0] : 0;
    };
    tp->o_half = half(tO);
    tp->v_half = half(tV);
    // Needed 8x8 output fragments per box triple and GEMM (the kernel's frag_needed: an 8-row half of
    // the row box x one p x 8 q holding some a<b<c inside the extents); the default kernel issues DMMAs
    // for these only.
    std::vector<std::array<int, 3>> nfrag(box3.size());
    for (size_t q = 0; q < box3.size(); ++q) {
      const int4 b3 = box3[q];
      const int32_t lo3[3] = {box_lo[b3.x], box_lo[b3.y], box_lo[b3.z]};
      const int32_t ex3[3] = {box_ext[b3.x], box_ext[b3.y], box_ext[b3.z]};
      for (int g = 0; g < 3; ++g) {
        int cnt = 0;
        for (int r0 = 0; r0 < kTripBox; r0 += 8)
          for (int col = 0; col < kTripBox * kTripBox; col += 8) {
            const int pp = col / kTripBox, q0 = col % kTripBox;
            int l[3], h[3];
            bool ok = true;
            for (int d = 0; d < 3 && ok; ++d) {
              int s0, e0;
              if (d == g) { s0 = r0; e0 = r0 + 8; }
              else if (d == (g == 0 ? 1 : 0)) { s0 = pp; e0 = pp + 1; }
              else { s0 = q0; e0 = q0 + 8; }
              const int hh = std::min(e0, (int)ex3[d]);
              ok = s0 < hh;
              l[d] = lo3[d] + s0;
              h[d] = lo3[d] + hh - 1;
            }
            if (!ok) continue;
            const int bb = std::max(l[0] + 1, l[1]);
            if (bb > h[1]) continue;
            if (std::max(bb + 1, l[2]) <= h[2]) ++cnt;
          }
        nfrag[q][g] = cnt;
      }
    }
    // per unit: stages of each GEMM (ceil(len / 8) per m / e segment; the segment ranges follow the
    // kernel's spin restriction) and the summed lengths of the non-zero products
    const int32_t oh = tp->o_half, vh = tp->v_half;
    auto so = [&](int32_t x) { return oh ? (x < oh ? 1 : -1) : 0; };
    auto sv = [&](int32_t v) { return vh ? (v < vh ? 1 : -1) : 0; };
    auto unit_stages = [&](int64_t q, int64_t st[3], int64_t& unit_len) {
      const int4 b3 = box3[units[q].x];
      const int4 tr = trip[units[q].y];
      const int32_t bl[3] = {box_lo[b3.x], box_lo[b3.y], box_lo[b3.z]};
      unit_len = 0;
      for (int g = 0; g < 3; ++g) {
        const int32_t sr = sv(bl[g]), sp = sv(g == 0 ? bl[1] : bl[0]), sq = sv(g == 2 ? bl[1] : bl[2]);
        st[g] = 0;
        for (int sg = 0; sg < 6; ++sg) {
          int64_t len;
          if (sg < 3) {
            const int32_t x = (sg == 2) ? tr.y : tr.x, y = (sg == 0) ? tr.y : tr.z;
            const int32_t sm = so(x) + so(y) - sr;
            len = !oh ? nO : (sm == 1 ? oh : (sm == -1 ? nO - oh : 0));
          } else {
            const int32_t x = (sg == 3) ? tr.x : (sg == 4 ? tr.y : tr.z);
            const int32_t se = sp + sq - so(x);
            len = !vh ? nV : (se == 1 ? vh : (se == -1 ? nV - vh : 0));
          }
          st[g] += (len + 7) / 8;
          unit_len += len;
        }
      }
    };
    // Cost-balanced contiguous ranges over the ranks: a unit costs its issued DMMA fragment-stages
    // (sum over the GEMMs of needed fragments x stages) plus a fixed per-unit share (prologue, three
    // folds, energy epilogue) of 3 x 64 + 256 -- diagonal box triples and spin-halved sums are cheaper.
    constexpr double kUnitFixed = 3.0 * 64.0 + 256.0;
    std::vector<double> cost((size_t)U);
    double cost_total = 0, cost_max = 0;
    for (int64_t q = 0; q < U; ++q) {
      int64_t st[3], ul;
      unit_stages(q, st, ul);
      const auto& nf = nfrag[units[q].x];
      cost[q] = (double)(nf[0] * st[0] + nf[1] * st[1] + nf[2] * st[2]) + kUnitFixed;
      cost_total += cost[q];
      cost_max = std::max(cost_max, cost[q]);
    }
    {
      // rank r takes the units whose cost midpoint falls in [C r / N, C (r + 1) / N)
      int64_t first = -1, last = -1;
      double acc = 0;
      const double lo_c = cost_total * (double)ctx->rank / (double)ctx->nranks;
      const double hi_c = cost_total * (double)(ctx->rank + 1) / (double)ctx->nranks;
      for (int64_t q = 0; q < U; ++q) {
        const double mid = acc + 0.5 * cost[q];
        acc += cost[q];
        if (mid >= lo_c && (mid < hi_c || ctx->rank == ctx->nranks - 1)) {
          if (first < 0) first = q;
          last = q;
        }
      }
      tp->unit0 = first < 0 ? 0 : first;
      tp->nunits = first < 0 ? 0 : last - first + 1;
    }
    // executed FLOPs of the default kernel: per unit and GEMM, the needed 8x8 fragments x stages of 8 k
    // rows (2 x 8 x 8 x 8 per fragment-stage)
    {
      double frag_stages = 0, rank_cost = 0;
      for (int64_t q = tp->unit0; q < tp->unit0 + tp->nunits; ++q) {
        int64_t st[3], ul;
        unit_stages(q, st, ul);
        const auto& nf = nfrag[units[q].x];
        frag_stages += (double)(nf[0] * st[0] + nf[1] * st[1] + nf[2] * st[2]);
        rank_cost += cost[q];
        alg += 2.0 * (double)ul * (double)box3_n[units[q].x];
      }
      (void)per;
      tp->info.flops_exec = frag_stages * 2.0 * 8.0 * 8.0 * 8.0;
      tp->info.cost_rank = rank_cost;
      tp->info.cost_total = cost_total;
      tp->info.cost_max_unit = cost_max;
    }
    tp->info.w_blocks_total = U;
    tp->info.w_blocks = tp->nunits;
    tp->info.batches = 1;
    tp->info.flops_alg = alg;
    // blocked copies of the default kernel (TriplesParams): after the partials
    {
      // padded summed rows: each spin range rounded up to a multiple of 8 (TriplesParams)
      auto pad8 = [](int64_t x) { return (x + 7) / 8 * 8; };
      tp->ko2 = (int32_t)pad8(tp->o_half);
      tp->kv2 = (int32_t)pad8(tp->v_half);
      tp->kpo = (int32_t)(tp->ko2 + pad8(nO - tp->o_half));
      tp->kpv = (int32_t)(tp->kv2 + pad8(nV - tp->v_half));
      const int64_t nbx = (int64_t)tp->nbox, o = nO, kpo = tp->kpo, kpv = tp->kpv;
      const int64_t ns[4] = {o * nbx * nbx * kpo * kTripBox * kTripBox, o * nbx * nbx * kpv * kTripBox * kTripBox,
                             o * o * nbx * kpo * kTripBox, o * o * nbx * kpv * kTripBox};
      int64_t pos = base + (U + 1) / 2 * 2;
      for (int q = 0; q < 4; ++q) {
        tp->blk_pos[q] = pos;
        tp->blk_n[q] = ns[q];
        pos += (ns[q] + 31) / 32 * 32;
      }
      base = pos - (U + 1) / 2 * 2;
    }
    tp->ws_need = base + (U + 1) / 2 * 2;
    tp->info.ws_elems = tp->ws_need;
    if (ctx->device >= 0) {
      TT_TRY(need_ws(ctx));
      DeviceGuard dg(ctx->device);
      for (int x = 0; x < 5; ++x) TT_TRY(build_retile(ctx, tp->rt[x]));
      TT_TRY(dev_alloc(ctx, tp->mem, &tp->d_units, std::max<size_t>(1, units.size())));
      TT_TRY(dev_alloc(ctx, tp->mem, &tp->d_box3, std::max<size_t>(1, box3.size())));
      TT_TRY(dev_alloc(ctx, tp->mem, &tp->d_trip, std::max<size_t>(1, trip.size())));
      TT_TRY(dev_alloc(ctx, tp->mem, &tp->d_box_lo, box_lo.size()));
      TT_TRY(dev_alloc(ctx, tp->mem, &tp->d_box_ext, box_ext.size()));
      if (!units.empty()) TT_CUDA(cudaMemcpy(tp->d_units, units.data(), units.size() * sizeof(int2), cudaMemcpyHostToDevice));
      // pairs of consecutive units of this rank with the same box triple, occupied pair (i,j) and spin of k
      // (then both units run the same segment ranges: the cluster kernel shares one operand per segment)
      std::vector<int2> pairs;
      const int32_t ohalf = tp->o_half;
      auto kspin = [&](int32_t k) { return ohalf ? (k < ohalf ? 1 : -1) : 0; };
      for (int64_t q = tp->unit0; q < tp->unit0 + tp->nunits;) {
        const bool two = q + 1 < tp->unit0 + tp->nunits && units[q + 1].x == units[q].x &&
                         trip[units[q + 1].y].x == trip[units[q].y].x && trip[units[q + 1].y].y == trip[units[q].y].y &&
                         kspin(trip[units[q + 1].y].z) == kspin(trip[units[q].y].z);
        pairs.push_back({(int)q, two ? 2 : 1});
        q += two ? 2 : 1;
      }
      tp->npairs = (int64_t)pairs.size();
      TT_TRY(dev_alloc(ctx, tp->mem, &tp->d_pairs, std::max<size_t>(1, pairs.size())));
      if (!pairs.empty()) TT_CUDA(cudaMemcpy(tp->d_pairs, pairs.data(), pairs.size() * sizeof(int2), cudaMemcpyHostToDevice));
      if (!box3.empty()) TT_CUDA(cudaMemcpy(tp->d_box3, box3.data(), box3.size() * sizeof(int4), cudaMemcpyHostToDevice));
      TT_CUDA(cudaMemcpy(tp->d_trip, trip.data(), trip.size() * sizeof(int4), cudaMemcpyHostToDevice));
      TT_CUDA(cudaMemcpy(tp->d_box_lo, box_lo.data(), box_lo.size() * 4, cudaMemcpyHostToDevice));
      TT_CUDA(cudaMemcpy(tp->d_box_ext, box_ext.data(), box_ext.size() * 4, cudaMemcpyHostToDevice));
    }
    plan_put(ctx, keybuf, tp);
  }
  if (info) *info = tp->info;
  if (!workspace) return TT_OK;   // query: units, FLOPs, workspace size
  if (!energy) return fail(TT_E_ARG, "NULL energy");
  if (!eps_o || !eps_v) return fail(TT_E_ARG, "NULL orbital energies");
  if (ws_elems < tp->ws_need)
    return fail(TT_E_OOM, "workspace holds %lld doubles, (T) needs %lld (dense input copies + one partial per unit)",
                (long long)ws_elems, (long long)tp->ws_need);
  TT_TRY(need_ws(ctx));
  for (int x = 0; x < 5; ++x) TT_TRY(check_bound(ins[x], names[x]));
  if (ctx->prepare_only) return TT_OK;
  DeviceGuard dg(ctx->device);
  reset_stats(ctx);
  double* ws = (double*)workspace;
  if ((uintptr_t)ws % 16) return fail(TT_E_ARG, "workspace must be 16-byte aligned");
  for (int x = 0; x < 5; ++x) {
    tp->rt[x].dst->data = ws + tp->rt[x].ws_pos;
    tp->rt[x].dst->capacity = tp->rt[x].dst->packed_elems;
    TT_TRY(run_retile(ctx, tp->rt[x]));
  }
  double* partials = ws + tp->rt[4].ws_pos + (tp->rt[4].dst->packed_elems + 31) / 32 * 32;
  TriplesParams p{};
  p.VO = tp->rt[0].dst->data;
  p.VV = tp->rt[1].dst->data;
  p.T2 = tp->rt[2].dst->data;
  p.VD = tp->rt[3].dst->data;
  p.T1 = tp->rt[4].dst->data;
  p.eps_o = eps_o;
  p.eps_v = eps_v;
  p.units = tp->d_units;
  p.box3 = tp->d_box3;
  p.trip = tp->d_trip;
  p.box_lo = tp->d_box_lo;
  p.box_ext = tp->d_box_ext;
  p.nO = (int32_t)nO;
  p.nV = (int32_t)nV;
  p.o_half = tp->o_half;
  p.v_half = tp->v_half;
  p.partials = partials;
  p.nb = tp->nbox;
  p.kpo = tp->kpo;
  p.kpv = tp->kpv;
  p.ko2 = tp->ko2;
  p.kv2 = tp->kv2;
  {   // blocked copies of the default kernel
    double* bq[4];
    for (int q = 0; q < 4; ++q) bq[q] = ws + tp->blk_pos[q];
    p.QT2 = bq[0];
    p.QVV = bq[1];
    p.PVO = bq[2];
    p.PT2 = bq[3];
    for (int q = 0; q < 4; ++q) {
      Launch L(ctx, "tt_triples_blockify");
      TT_CUDA(launch_blockify(q, p, bq[q], tp->blk_n[q], ctx->stream));
    }
  }
  // bulk copies of the blocked operands (default), TMA boxes (opt-in pair / cluster kernels) or cp.async
  // staging (TT_TMA=0)
  const char* ft = getenv("TT_TMA");
  const bool use_tma = !ft || atoi(ft) != 0;
  CUtensorMap maps[4];
  if (use_tma) {
    const uint32_t bP[4] = {(uint32_t)kTripBox + 4, 8, 1, 1}, bQ[4] = {(uint32_t)kTripBox + 2, (uint32_t)kTripBox + 2, 1, 8};
    const int64_t dVO[4] = {nV, nO, nO, nO}, dT2[4] = {nV, nV, nO, nO}, dVV[4] = {nV, nV, nO, nV};
    TT_TRY(encode_4d(&maps[0], p.VO, dVO, bP));
    TT_TRY(encode_4d(&maps[1], p.T2, dT2, bP));
    TT_TRY(encode_4d(&maps[2], p.T2, dT2, bQ));
    TT_TRY(encode_4d(&maps[3], p.VV, dVV, bQ));
  }
  // opt-in: the 2-CTA cluster kernel with TMA multicast of the shared operand (TT_TRIPLES_CLUSTER=1;
  // measured 5.79 s vs 3.08 s at O=40 V=200: the two CTAs release every slot together, so each waits on
  // the other's slowest warp) or the 16-warp pair kernel (TT_TRIPLES_PAIR=1; 4.59 s)
  const char* fp = getenv("TT_TRIPLES_PAIR");
  const char* fc = getenv("TT_TRIPLES_CLUSTER");
  const bool use_pair = use_tma && fp && atoi(fp) != 0;
  const bool use_cluster = use_tma && !use_pair && fc && atoi(fc) != 0;
  ctx->last.producer = use_pair ? 2 : (use_cluster ? 3 : (use_tma ? 1 : 0));
  if (use_pair || use_cluster) {
    for (int64_t q0 = 0; q0 < tp->npairs; q0 += (1 << 20)) {
      p.pairs = tp->d_pairs + q0;
      Launch L(ctx, "tt_triples_fused");
      const int64_t np = std::min<int64_t>(1 << 20, tp->npairs - q0);
      if (use_cluster) TT_CUDA(launch_triples_cluster(p, maps, np, ctx->stream));
      else TT_CUDA(launch_triples_pair(p, maps, np, ctx->stream));
    }
  }
  // launches of at most 2^20 units (keeps each launch's grid small; partials are indexed by unit)
  for (int64_t u0 = tp->unit0; !use_pair && !use_cluster && u0 < tp->unit0 + tp->nunits; u0 += (1 << 20)) {
    p.unit0 = u0;
    const int64_t n = std::min<int64_t>(1 << 20, tp->unit0 + tp->nunits - u0);
    Launch L(ctx, "tt_triples_fused");
    if (use_tma) TT_CUDA(launch_triples_tma(p, maps, n, ctx->stream));
    else TT_CUDA(launch_triples_fused(p, n, ctx->stream));
  }
  {
    Launch L(ctx, "tt_scalar_final");
    TT_CUDA(launch_scalar_final(partials + tp->unit0, tp->nunits, 1.0, ctx->d_scalar, nullptr, ctx->stream));
  }
  TT_TRY(allreduce_sum(ctx, ctx->d_scalar, ctx->stream));
  TT_CUDA(cudaMemcpyAsync(energy, ctx->d_scalar, 8, cudaMemcpyDeviceToHost, ctx->stream));
  TT_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->last.c_blocks = tp->nunits;
  ctx->last.flops = tp->info.flops_alg;
  ctx->last.aux_flops = tp->info.flops_exec;
  return TT_OK;
}

}  // extern "C"
