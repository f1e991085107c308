// tt_cholesky.cpp -- contraction with an implicit Cholesky-factored operand (PAPER Eq. cc12, P312-318).  Citations as in include/tt.h.
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
// When the workspace also holds BsT(s,r,..) = Bs(r,s,..) (TT_CHOL_BST != 0) pass 2 reads
//   - sum W(p,q,s,r) BsT(s,r)   (both operands in K order (s,r): TMA-eligible, unlike W(p,q,s,r) Bs(r,s)).
// When the workspace cannot hold Bh plus one W row (or TT_CHOL_TWO_PASS=1) the consume reads B
// directly in two passes, C += alpha W.B and C -= alpha W.B(r<->s): no Bh, twice the consume FLOPs.

namespace tt {

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
  tt_tensor BsT = nullptr;                      // Bs with r and s swapped (K order of W read as (p,q,s,r))
  std::shared_ptr<ElemPlan> t_plan;             // BsT formation from Bh
  bool use_t = false;                           // exchange consume on BsT (TMA-eligible) instead of Bs
  std::shared_ptr<ContractPlan> vplan, wplan;   // SPMD plans: this rank's C parts, FLOP counts
  std::shared_ptr<ElemPlan> copy_plan, swap_plan;   // Bh formation (this rank's Bh blocks)
  GatherPlan bgather;                           // all-gather of B (not co-located) ...
  GatherPlan hgather;                           // ... or of Bh (co-located B pairs)
  GatherPlan xgather;                           // nranks > 1: the blocks of X this rank does not hold
  std::vector<CholBatch> batches;
  std::string lc;                               // the auxiliary label used for L
  bool two_pass = false;                        // no room for Bh: consume W.B and W.B(r<->s)
  bool colocated = false;
  ~CholPlan() {
    delete Vmeta;
    delete Wmeta;
    delete Bh;
    delete Bs;
    delete BsT;
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

}  // namespace tt

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
  if (ctx->nranks > 1 && X->compact)
    return fail(TT_E_UNSUPPORTED, "with nranks > 1 the Cholesky vectors X need their full packed storage "
                "(not compact): every rank builds W from all of X");
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
    // BsT(s,r,..) = Bs(r,s,..): the exchange consume -W(p,q,s,r) Bs(r,s,..) then reads both operands
    // in the same K order (s,r), which the TMA producer can stage (Bs's order against W's cannot)
    {
      std::vector<uint8_t> tnz(B->nblocks, 0);
      for (int64_t x = 0; x < B->nblocks; ++x)
        if (snz[x]) tnz[swap_of[x]] = 1;
      TT_TRY(new_meta_tensor(ctx, B->dims, tnz, &cp->BsT));
      for (int64_t x = 0; x < B->nblocks; ++x)
        if (tnz[x]) cp->BsT->owner[x] = TT_REPLICATED;
    }
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
    if (ctx->nranks > 1) {   // owner-distributed X: every rank builds W from all of X
      Needs nx(ctx->nranks);
      for (int rr = 0; rr < ctx->nranks; ++rr)
        for (int64_t x = 0; x < X->nblocks; ++x)
          if (X->nz[x]) nx[rr].push_back({0, x, 0, X->block_volume(x)});
      TT_TRY(build_gather(ctx, nx, {X}, cp->xgather));
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
    std::vector<int64_t> rb, uels;
    int64_t max_uel = 0;
    for (auto& kv : units) {
      row_blocks(kv.second, rb);
      int64_t uel = 0;
      for (int64_t vb : rb) uel += (cp->Wmeta->block_volume(vb) + 1) / 2 * 2;
      max_uel = std::max(max_uel, uel);
      uels.push_back(uel);
    }
    auto n_batches = [&](int64_t cap) {   // the greedy packing of flush() below
      int64_t n = 0, cur = 0;
      for (int64_t u : uels) {
        if (cur > 0 && cur + u > cap) { ++n; cur = 0; }
        cur += u;
      }
      return n + (cur > 0 ? 1 : 0);
    };
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
    // BsT after Bh when the workspace still holds a W row after both and the smaller W space adds at
    // most half again as many batches (smaller batches lose more to tails than the TMA consume gains:
    // configs[3]-scale ladder in 40 GB 29 -> 43 batches, 2 % faster; the CCSD iteration's ladder in
    // 12 GB 86 -> 256 batches, 3 % slower).  TT_CHOL_BST=0: off, =1: whenever it fits.
    const int64_t bst_elems = (cp->BsT->packed_elems + 31) / 32 * 32;
    const char* fb = getenv("TT_CHOL_BST");
    const int bst_mode = fb ? atoi(fb) : 2;
    cp->use_t = !cp->two_pass && bst_mode != 0 && cp->BsT->packed_elems > 0 &&
                ws_elems >= bh_elems + bst_elems + max_uel &&
                (bst_mode == 1 || 2 * n_batches(ws_elems - bh_elems - bst_elems) <= 3 * n_batches(ws_elems - bh_elems));
    if (cp->use_t) {
      cp->BsT->data = (double*)workspace + bh_elems;
      cp->BsT->capacity = bst_elems;
      TT_TRY(local_add_plan(ctx, cp->BsT, cp->Bs, sw, 0.0, cp->t_plan));
    }
    const int64_t w_off = cp->two_pass ? 0 : bh_elems + (cp->use_t ? bst_elems : 0);
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
  tt_tensor xB = cp->use_t ? cp->BsT : cp->Bs;                                        // exchange operand
  const char* xl = cp->use_t ? bsw.c_str() : bl;                                      // ... and its labels
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
        TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vsw.c_str(), xB, xl, 1.0, px, &dummy, bt.copt));
      }
    }
    return TT_OK;
  }
  reset_stats(ctx);
  trace("cholesky: plans ready, batches", (long long)cp->batches.size());
  trace("cholesky: exchange consume on BsT", cp->use_t ? 1 : 0);
  TT_TRY(run_gather(ctx, cp->xgather, {X}));
  TT_TRY(run_gather(ctx, cp->bgather, {B}));
  trace("B gathered, runs", (long long)(cp->bgather.recv.size() + cp->bgather.send.size()));
  if (!cp->two_pass) {
    TT_TRY(run_local_add(ctx, *cp->copy_plan, cp->Bh, B, 0.0, 1.0));
    TT_TRY(run_local_add(ctx, *cp->swap_plan, cp->Bh, B, 1.0, -1.0));
    trace("Bh formed");
    TT_TRY(run_gather(ctx, cp->hgather, {cp->Bh}));
    trace("Bh gathered, runs", (long long)(cp->hgather.recv.size() + cp->hgather.send.size()));
    if (cp->use_t) TT_TRY(run_local_add(ctx, *cp->t_plan, cp->BsT, cp->Bs, 0.0, 1.0));
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
      TT_TRY(get_contract_plan(ctx, C, cl, bt.Wb, vsw.c_str(), xB, xl, 1.0, px, &dummy, bt.copt));
      TT_TRY(launch_plan(ctx, *pu, C, cl, beta, alpha, bt.Wb, vl, cp->Bh, bl));
      TT_TRY(launch_plan(ctx, *px, C, cl, 1.0, -alpha, bt.Wb, vsw.c_str(), xB, xl));
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
