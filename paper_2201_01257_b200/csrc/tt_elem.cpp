// tt_elem.cpp -- element operations (set / add / fill / scalar): per-descriptor kernel modes, segment lists.  Citations as in include/tt.h.
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
// element operations (set / add / fill / scalar): segment lists built on the host

namespace tt {



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


void reset_stats(tt_ctx ctx) { ctx->last = tt_stats{}; }

}  // namespace tt

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
