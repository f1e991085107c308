// tt_triples_host.cpp -- perturbative triples (T) host side: plan, re-tiling, blocking, launches (PAPER Eqs. cc14,
// tensort, abt, tensort2, P343-413).  Citations as in include/tt.h.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
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
  GatherPlan gp;                              // nranks > 1: every input block this rank does not hold
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
    if (ctx->nranks > 1 && ins[x]->compact)
      return fail(TT_E_UNSUPPORTED, "%s: with nranks > 1 the inputs need their full packed storage (not compact): "
                  "every rank reads all of them", names[x]);
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
    if (ctx->nranks > 1) {   // owner-distributed inputs: every rank receives all blocks it does not hold
      Needs need(ctx->nranks);
      for (int r = 0; r < ctx->nranks; ++r)
        for (int x = 0; x < 5; ++x)
          for (int64_t b = 0; b < ins[x]->nblocks; ++b)
            if (ins[x]->nz[b]) need[r].push_back({x, b, 0, ins[x]->block_volume(b)});
      TT_TRY(build_gather(ctx, need, {ins[0], ins[1], ins[2], ins[3], ins[4]}, tp->gp));
    }
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
  TT_TRY(run_gather(ctx, tp->gp, {ins[0], ins[1], ins[2], ins[3], ins[4]}));
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
  // bulk copies of the blocked operands (default), TMA boxes (opt-in pair / cluster kernels) or cp.async
  // staging (TT_TMA=0).  Opt-in: the 2-CTA cluster kernel with TMA multicast of the shared operand
  // (TT_TRIPLES_CLUSTER=1; measured 5.79 s vs 3.08 s at O=40 V=200: the two CTAs release every slot
  // together, so each waits on the other's slowest warp) or the 16-warp pair kernel (TT_TRIPLES_PAIR=1;
  // 4.59 s)
  const char* ft = getenv("TT_TMA");
  const bool use_tma = !ft || atoi(ft) != 0;
  const char* fp = getenv("TT_TRIPLES_PAIR");
  const char* fc = getenv("TT_TRIPLES_CLUSTER");
  const bool use_pair = use_tma && fp && atoi(fp) != 0;
  const bool use_cluster = use_tma && !use_pair && fc && atoi(fc) != 0;
  if (use_tma && !use_pair && !use_cluster) {   // blocked copies of the default kernel
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
  CUtensorMap maps[4];
  if (use_pair || use_cluster) {   // 4-D TMA boxes over the dense copies
    const uint32_t bP[4] = {(uint32_t)kTripBox + 4, 8, 1, 1}, bQ[4] = {(uint32_t)kTripBox + 2, (uint32_t)kTripBox + 2, 1, 8};
    const int64_t dVO[4] = {nV, nO, nO, nO}, dT2[4] = {nV, nV, nO, nO}, dVV[4] = {nV, nV, nO, nV};
    TT_TRY(encode_4d(&maps[0], p.VO, dVO, bP));
    TT_TRY(encode_4d(&maps[1], p.T2, dT2, bP));
    TT_TRY(encode_4d(&maps[2], p.T2, dT2, bQ));
    TT_TRY(encode_4d(&maps[3], p.VV, dVV, bQ));
  }
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
    if (use_tma) TT_CUDA(launch_triples_tma(p, n, ctx->stream));
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
