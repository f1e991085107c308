// tt_contract.cpp -- contraction: plans (variant, producer, work items, split-K), execution, the host-buffer
// call, task lists, partitions and gather plans.  Citations as in include/tt.h.
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
// contraction

namespace tt {


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
                              const ContractOpts& opts) {
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
  // Wave tail (TT_TAIL_SPLIT=0: off).  With W work items on S = SMs x CTAs/SM resident slots the last
  // W mod S items run while the other slots idle; when they fit one per SM after re-tiling with the
  // smallest warp-specialised tile, they form a second launch of that variant over narrowed copies of
  // their groups (same tasks, same per-element k order: bitwise the same C, R12), which takes a fraction
  // of a full wave instead of a whole one.
  {
    const char* ft = getenv("TT_TAIL_SPLIT");
    int tv = -1;
    if ((!ft || atoi(ft) != 0) && pl.splits.empty() && pl.variant >= num_contract_variants()) {
      auto area = [](const VariantInfo& x) { return (int64_t)x.bm * x.bn; };
      for (int v = num_contract_variants(); v < n_variants(); ++v)
        if (area(variant_info(v)) < area(vi) && (tv < 0 || area(variant_info(v)) < area(variant_info(tv)))) tv = v;
    }
    if (tv >= 0) {
      const VariantInfo tvi = variant_info(tv);
      int64_t slots = (int64_t)ctx->sm_count * std::max(vi.ctas_per_sm, 1);
      if (const char* fs = getenv("TT_TAIL_SLOTS")) slots = std::max<int64_t>(1, atoll(fs));   // tests
      const int64_t W = (int64_t)work.size(), r = W % slots;
      const int64_t per = ((int64_t)vi.bm / tvi.bm + (vi.bm % tvi.bm != 0)) * ((int64_t)vi.bn / tvi.bn + (vi.bn % tvi.bn != 0));
      if (getenv("TT_DEBUG") && atoi(getenv("TT_DEBUG")) != 0)
        fprintf(stderr, "[tt rank %d] wave tail: %lld items, %lld slots, remainder %lld x %lld tail tiles, variant %d -> %d\n",
                ctx->rank, (long long)W, (long long)slots, (long long)r, (long long)per, pl.variant, tv);
      if (W > slots && r > 0 && r * per <= std::max<int64_t>(ctx->sm_count, 1)) {
        std::vector<CGroupDesc> tg;
        std::vector<WorkItem> tw;
        for (int64_t i = W - r; i < W; ++i) {
          const WorkItem& w = work[i];
          CGroupDesc g = groups[w.group];
          g.m_begin = groups[w.group].m_begin + w.mt * vi.bm;
          g.M = std::min<int32_t>(groups[w.group].M, g.m_begin + vi.bm);
          g.n_begin = groups[w.group].n_begin + w.nt * vi.bn;
          g.N = std::min<int32_t>(groups[w.group].N, g.n_begin + vi.bn);
          const int32_t gi = (int32_t)tg.size();
          tg.push_back(g);
          for (int32_t mt = 0; mt < (g.M - g.m_begin + tvi.bm - 1) / tvi.bm; ++mt)
            for (int32_t nt = 0; nt < (g.N - g.n_begin + tvi.bn - 1) / tvi.bn; ++nt) tw.push_back({gi, mt, nt});
        }
        work.resize(W - r);
        TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_tail_groups, tg.size()));
        TT_TRY(dev_alloc(ctx, pl.mem, &pl.d_tail_work, tw.size()));
        TT_CUDA(cudaMemcpy(pl.d_tail_groups, tg.data(), tg.size() * sizeof(CGroupDesc), cudaMemcpyHostToDevice));
        TT_CUDA(cudaMemcpy(pl.d_tail_work, tw.data(), tw.size() * sizeof(WorkItem), cudaMemcpyHostToDevice));
        pl.tail_variant = tv;
        pl.tail_nwork = (int64_t)tw.size();
      }
    }
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
                            const ContractOpts& opts) {
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
  if (pl.tail_nwork > 0) {   // the wave tail on the smallest tile (see build_contract_plan)
    Launch L(ctx, nm.c_str());
    ContractParams q = p;
    q.groups = pl.d_tail_groups;
    q.work = pl.d_tail_work;
    q.nwork = pl.tail_nwork;
    q.persistent = 0;
    const int tv = pl.tail_variant - num_contract_variants();
    if (pl.tma) {
      ContractPlan& mp = const_cast<ContractPlan&>(pl);
      if (mp.tail_map_ptr[0] != A->data || mp.tail_map_ptr[1] != B->data) {
        const VariantInfo vt = variant_info(pl.tail_variant);
        TT_TRY(encode_2d(&mp.tail_maps[0], A->data, pl.tma_k, A->storage_elems / pl.tma_k, 16, (uint32_t)vt.bm, true));
        if (pl.tma_mode & 1) {
          TT_TRY(encode_2d(&mp.tail_maps[1], B->data, pl.tma_n, B->storage_elems / pl.tma_n, 16, (uint32_t)vt.bn, true));
        } else {
          const int64_t d3[3] = {pl.tma_n, pl.tma_k, B->storage_elems / (pl.tma_n * pl.tma_k)};
          const uint32_t b3[3] = {(uint32_t)vt.bn + 2, 16, 1};
          TT_TRY(encode_3d(&mp.tail_maps[1], B->data, d3, b3));
        }
        mp.tail_map_ptr[0] = A->data;
        mp.tail_map_ptr[1] = B->data;
      }
      TT_CUDA(launch_contract_tma(tv, pl.tma_mode, q, pl.tail_maps, pl.tail_nwork, ctx->stream));
    } else {
      TT_CUDA(launch_contract_ws(tv, pl.an.a_kc, pl.an.b_nc, pl.a_vec, pl.b_vec, q, pl.tail_nwork, ctx->stream));
    }
  }
  if (!pl.splits.empty()) {
    const std::string rn = std::string("tt_contract_reduce[") + cl + "=" + al + "*" + bl + "]";
    Launch R(ctx, rn.c_str());
    TT_CUDA(launch_split_reduce(pl.d_partials, C->data, pl.d_groups, pl.d_splits, (int32_t)pl.splits.size(),
                                p.nM, p.nN, alpha, beta, ctx->stream));
  }
  return TT_OK;
}

}  // namespace tt

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

// End to end from host memory (tt.h tt_contract_host).  Pipelined (A's and C's dim 0 carry the same label
// on the same tiling, no views; with several ranks A's rows local to the rank's C rows, B's remote
// blocks gathered once up front): per chunk x of C -- the blocks sharing C's dim-0 tile,
// or its (dim-0, dim-1) tile pair when dim 0 has fewer than kHostMinChunks tiles and A's dim 1 carries
// C's dim-1 label -- A's blocks with the same leading coordinates (one contiguous packed range,
// row-major block order) go host->device on the context's copy stream while chunk x-1 contracts; chunk
// x is a local plan restricted to its C blocks (the same per-element k order as the whole contraction:
// bitwise the same result, R12); its C rows go device->host while chunk x+1 contracts.  Otherwise: H2D
// of every held range, tt_contract, D2H of this rank's C ranges.
namespace {
struct HostPlan {
  bool pipelined = false;
  int32_t lead = 1;   // leading dims of C (shared with A) that define a pipeline chunk: 1 or 2
  int32_t nt1 = 1;    // tiles of C's dim 1 when lead == 2
  std::vector<std::vector<std::pair<int64_t, int64_t>>> a_rng, c_rng;   // per chunk: held storage of A, C
  std::vector<std::shared_ptr<ContractPlan>> tiles;        // local plan of each chunk (nullptr: no C block)
  int32_t chunk(const int32_t* co) const { return lead == 2 ? co[0] * nt1 + co[1] : co[0]; }
};

// chunks of the host pipeline: finer chunks shorten the exposed first upload and last contraction;
// dims 0 and 1 are used together when dim 0 alone gives fewer than this many
constexpr int32_t kHostMinChunks = 16;

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
    // with several ranks, A's rows must be local to this rank's C rows (no gather entry of A): B's gather
    // runs once up front, A arrives chunk by chunk
    bool a_local = true;
    if (A != B)
      for (const auto* lst : {&whole->gp.send_list, &whole->gp.recv_list})
        for (size_t i = 0; i + 4 < lst->size(); i += 5) a_local = a_local && (*lst)[i] != 0;
    hp->pipelined = same0 && a_local && !A->view_of && !C->view_of && A != B && !C->compact;
    if (hp->pipelined) {
      // blocks sharing C's (and A's) leading block coordinates are contiguous in packed order; each
      // chunk moves this rank's held ranges of those blocks
      const bool two = C->order >= 2 && A->order >= 2 && C->dims[0]->ntiles() < kHostMinChunks && al[1] == cl[1] &&
                       same_tiling(A->dims[1], C->dims[1]);
      hp->lead = two ? 2 : 1;
      hp->nt1 = two ? C->dims[1]->ntiles() : 1;
      const int32_t nt = C->dims[0]->ntiles() * hp->nt1;
      hp->a_rng.assign(nt, {});
      hp->c_rng.assign(nt, {});
      hp->tiles.assign(nt, nullptr);
      int32_t co[TT_MAX_ORDER];
      std::vector<std::pair<int64_t, int64_t>> hr;
      auto held = [&](tt_tensor T, std::vector<std::vector<std::pair<int64_t, int64_t>>>& rng) {
        for (int64_t b = 0; b < T->nblocks; ++b) {
          if (!T->nz[b] || T->blk_off[b] < 0) continue;
          T->block_coords(b, co);
          auto& v = rng[hp->chunk(co)];
          T->held_ranges(b, ctx->rank, hr);
          for (auto& h : hr) {
            const int64_t a0 = T->blk_off[b] + h.first, a1 = T->blk_off[b] + h.second;
            if (!v.empty() && a0 - v.back().second <= 1) v.back().second = std::max(v.back().second, a1);
            else v.push_back({a0, a1});
          }
        }
      };
      held(A, hp->a_rng);
      held(C, hp->c_rng);
      // each chunk's plan: this rank's parts of the chunk's C blocks (the whole plan's owner-computes rows)
      std::vector<std::vector<PartSel>> sel(nt);
      for (const auto& mp : whole->my) {
        const int64_t cb = whole->ht.cblk[mp.g];
        C->block_coords(cb, co);
        sel[hp->chunk(co)].push_back({cb, mp.lo, mp.hi});
      }
      for (int32_t x = 0; x < nt; ++x) {
        if (sel[x].empty()) continue;
        ContractOpts o;
        o.local = true;
        o.tag = "|host" + std::to_string(x);
        o.sel = std::move(sel[x]);
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
    TT_TRY(h2d(A, hA, hp->a_rng[x], ctx->copy_stream));
    TT_CUDA(cudaEventRecord(up[x], ctx->copy_stream));
  }
  // B's remote parts (several ranks) while A streams in; the chunk plans are local
  TT_TRY(run_gather(ctx, whole->gp, {A, B}));
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
      TT_TRY(d2h(C, hC, hp->c_rng[x], ctx->copy_stream));
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
