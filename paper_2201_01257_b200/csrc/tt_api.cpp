// tt_api.cpp -- host side of libtt, part 1: error state, the device workspace (arena, retired
// regions, plan cache eviction), contexts and simulated ranks, index spaces, tiled index spaces and
// tensors (layout, owners, parts, views, binding), plus the shared helpers declared in tt_host.h
// (label analysis, task enumeration, the gather).  The other C ABI calls live in tt_elem.cpp,
// tt_contract.cpp, tt_cholesky.cpp, tt_contract3.cpp and tt_triples_host.cpp.  Citations as in tt.h.
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
#include "tt_host.h"


using namespace tt;

namespace tt {

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

}  // namespace tt

tt_status tt::set_error(tt_status code, const char* msg) { return fail(code, "%s", msg); }

namespace tt {




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

}  // namespace tt

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

namespace tt {


tt_status nccl_check(int r, const char* what) {
  if (r == 0) return TT_OK;
  const char* err = nullptr;
  const NcclApi* api = nccl_api(&err);
  return fail(TT_E_NCCL, "%s failed: %s", what, api && api->GetErrorString ? api->GetErrorString(r) : "?");
}


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
                     cudaStream_t stream) {
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



std::string plan_key(const char* kind, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                     const char* bl, double beta) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s|%llu.%llu|%llu.%llu|%llu.%llu|%s|%s|%s|%d", kind, (unsigned long long)C->uid,
           (unsigned long long)C->version, (unsigned long long)A->uid, (unsigned long long)A->version,
           (unsigned long long)(B ? B->uid : 0), (unsigned long long)(B ? B->version : 0), cl, al, bl ? bl : "",
           beta != 0.0);
  return buf;
}

}  // namespace tt

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

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// tensors

// a view copies its parent's block map, storage offsets and owners at creation: the parent's layout
// may not change while views of it exist (they would keep stale offsets and owners)
tt_status tt::check_no_views(tt_tensor t) {
  if (t->live_views > 0)
    return fail(TT_E_STATE, "tensor has %d live view(s): destroy them before changing its layout", t->live_views);
  return TT_OK;
}

tt_status tt::tensor_new(tt_ctx ctx, int32_t order, const tt_tis* dims, tt_tensor* out) {
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

void tt::tensor_finish(tt_tensor t) {
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
void tt::apply_storage(tt_tensor t) {
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

void tt::refresh_parts_view(tt_tensor t) {
  t->pv_blk.clear(); t->pv_lo.clear(); t->pv_hi.clear(); t->pv_owner.clear();
  t->any_split = false;
  for (int64_t b = 0; b < t->nblocks; ++b) {
    for (const auto& p : t->parts[b]) {
      t->pv_blk.push_back(b); t->pv_lo.push_back(p.lo); t->pv_hi.push_back(p.hi); t->pv_owner.push_back(p.owner);
      t->any_split = true;
    }
  }
}

extern "C" {

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
