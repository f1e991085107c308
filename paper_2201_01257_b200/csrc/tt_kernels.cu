// tt_kernels.cu -- sm_100a kernels of libtt.
//
//  * tt_contract_kernel   block-sparse grouped FP64 GEMM: one CTA per work item
//                         (non-zero C block, BM x BN sub-tile); K loop over the block's task list
//                         (non-zero A/B tile pairs, P111/P138/P210) and, inside each task, over BK
//                         slices.  Operands are staged global -> shared memory by cp.async (LDGSTS)
//                         straight from their NATIVE block layout: the index permutation of each
//                         operand (TAMM's separate HPTT/LibreTT transpose, P107/P220) is folded into
//                         the per-element source address (label-group strides), so no transposed copy
//                         is ever written to HBM.  The math is FP64 tensor-core MMA (mma.sync m8n8k4
//                         -> DMMA.8x8x4 on sm_100a; tcgen05 has no f64 kind), accumulated in registers
//                         over all pairs of the block in canonical task order (deterministic, no
//                         atomics, reading R12).  Epilogue C = beta*C + alpha*acc with the output
//                         permutation (P172-174).
//  * build_count / build_scan / build_fill   device task-list builder (A2): count -> scan -> fill.
//  * set / add / fill / scalar               element kernels (A8-A10, synthetic inputs).
#include <cstdint>
#include <cstdio>

#include "tt_launch.h"

namespace tt {

// ------------------------------------------------------------------------------------------------
// small device helpers

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 8 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Mixed-radix decode of idx over n groups (innermost last) dotted with strides.
__device__ __forceinline__ int32_t dot_decode(int32_t idx, int n, const int32_t* ext, const int32_t* str) {
  int32_t off = 0;
#pragma unroll
  for (int g = kMaxGroup - 1; g > 0; --g) {
    if (g < n) {
      int32_t q = idx / ext[g];
      off += (idx - q * ext[g]) * str[g];
      idx = q;
    }
  }
  return off + idx * str[0];
}

// ------------------------------------------------------------------------------------------------
// Contraction kernel

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MINB_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int NW = WM * WN, NTHREADS = NW * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int MT = WTM / 8, NT = WTN / 8;
  static constexpr int KG = BK / 4;        // groups of 4 k values (one 8x4 / 4x8 copy patch each)
  static constexpr int MSTEP = NW / KG;    // warps sharing one k group
  static constexpr int RA = (BM / 8) / MSTEP;
  static constexpr int RB = (BN / 8) / MSTEP;
  static constexpr int LDA = BM + 8, LDB = BN + 8;   // row stride = 64 B mod 128 B: conflict-free
  static constexpr int SMEM = STAGES * BK * (LDA + LDB) * 8 + 256;
  static_assert(NW % KG == 0, "warps must cover the k groups");
  static_assert((BM / 8) % MSTEP == 0 && (BN / 8) % MSTEP == 0, "patch split");
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile");
};

template <class K, bool A_KC, bool B_NC>
__global__ void __launch_bounds__(K::NTHREADS, K::MINB) tt_contract_kernel(const ContractParams p) {
  extern __shared__ __align__(128) double smem[];
  double* sA = smem;
  double* sB = smem + K::STAGES * K::BK * K::LDA;
  __shared__ CGroupDesc g;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const WorkItem w = p.work[blockIdx.x];
  if (tid == 0) g = p.groups[w.group];
  __syncthreads();

  const int m0 = g.m_begin + w.mt * K::BM, n0 = g.n_begin + w.nt * K::BN;
  const int M = g.M, N = g.N;
  const int nM = p.nM, nN = p.nN, nK = p.nK;

  // ---- copy mapping: warp -> k group kq (4 consecutive k), patches of 8 rows x 4 k
  const int kq = warp % K::KG, mp0 = warp / K::KG;
  const int a_kl = A_KC ? (lane & 3) : (lane >> 3);
  const int a_rl = A_KC ? (lane >> 2) : (lane & 7);
  const int b_kl = B_NC ? (lane >> 3) : (lane & 3);
  const int b_rl = B_NC ? (lane & 7) : (lane >> 2);
  const int a_k = 4 * kq + a_kl, b_k = 4 * kq + b_kl;

  // ---- loader state (uniform task cursor; per-thread row offsets)
  int t_cur = g.task_begin, t_end = g.task_end, k0 = 0;
  const double* a_ptr = p.A;
  const double* b_ptr = p.B;
  int32_t Kt = 0;
  int32_t kext[kMaxGroup], akst[kMaxGroup], bkst[kMaxGroup];
  int32_t offAm[K::RA], offBn[K::RB];

  auto setup_task = [&](int t) {
    const TaskDesc* td = p.tasks + t;
    a_ptr = p.A + td->a_off;
    b_ptr = p.B + td->b_off;
    Kt = td->K;
    int32_t amst[kMaxGroup], bnst[kMaxGroup];
#pragma unroll
    for (int i = 0; i < kMaxGroup; ++i) {
      kext[i] = td->kext[i];
      akst[i] = td->ak_str[i];
      bkst[i] = td->bk_str[i];
      amst[i] = td->am_str[i];
      bnst[i] = td->bn_str[i];
    }
#pragma unroll
    for (int i = 0; i < K::RA; ++i) {
      int m = m0 + 8 * (mp0 + K::MSTEP * i) + a_rl;
      offAm[i] = (m < M) ? dot_decode(m, nM, g.mext, amst) : -1;
    }
#pragma unroll
    for (int i = 0; i < K::RB; ++i) {
      int n = n0 + 8 * (mp0 + K::MSTEP * i) + b_rl;
      offBn[i] = (n < N) ? dot_decode(n, nN, g.next, bnst) : -1;
    }
  };
  if (t_cur < t_end) setup_task(t_cur);

  auto load_stage = [&](int slot) {
    if (t_cur >= t_end) return;
    {
      const int k = k0 + a_k;
      const bool kv = k < Kt;
      const int32_t offk = kv ? dot_decode(k, nK, kext, akst) : 0;
      double* dst = sA + (slot * K::BK + a_k) * K::LDA;
#pragma unroll
      for (int i = 0; i < K::RA; ++i) {
        const bool v = kv && offAm[i] >= 0;
        cp_async8(dst + 8 * (mp0 + K::MSTEP * i) + a_rl, v ? (const void*)(a_ptr + offAm[i] + offk) : (const void*)p.A, v);
      }
    }
    {
      const int k = k0 + b_k;
      const bool kv = k < Kt;
      const int32_t offk = kv ? dot_decode(k, nK, kext, bkst) : 0;
      double* dst = sB + (slot * K::BK + b_k) * K::LDB;
#pragma unroll
      for (int i = 0; i < K::RB; ++i) {
        const bool v = kv && offBn[i] >= 0;
        cp_async8(dst + 8 * (mp0 + K::MSTEP * i) + b_rl, v ? (const void*)(b_ptr + offBn[i] + offk) : (const void*)p.B, v);
      }
    }
    k0 += K::BK;
    if (k0 >= Kt) {
      k0 = 0;
      ++t_cur;
      if (t_cur < t_end) setup_task(t_cur);
    }
  };

  // ---- accumulators
  const int wm = warp / K::WN, wn = warp % K::WN;
  double acc[K::MT][K::NT][2];
#pragma unroll
  for (int i = 0; i < K::MT; ++i)
#pragma unroll
    for (int j = 0; j < K::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nst = g.nstages;
#pragma unroll
  for (int s = 0; s < K::STAGES - 1; ++s) {
    load_stage(s);
    cp_async_commit();
  }

  const int fr_k = lane & 3, fr_r = lane >> 2;
  for (int s = 0; s < nst; ++s) {
    cp_async_wait<K::STAGES - 2>();
    __syncthreads();
    load_stage((s + K::STAGES - 1) % K::STAGES);
    cp_async_commit();
    const double* a = sA + (s % K::STAGES) * K::BK * K::LDA + wm * K::WTM + fr_r;
    const double* b = sB + (s % K::STAGES) * K::BK * K::LDB + wn * K::WTN + fr_r;
#pragma unroll
    for (int kk = 0; kk < K::BK / 4; ++kk) {
      // k of this lane in DMMA step kk: the two steps of every 8-wide k octet take k = 2*(lane%4) + t,
      // the grouping of the warp-specialised family, so that every variant adds each output element's
      // products in the same groups of four (identical bits across variants, R12)
      const int kr = 8 * (kk >> 1) + 2 * fr_k + (kk & 1);
      double af[K::MT], bf[K::NT];
#pragma unroll
      for (int i = 0; i < K::MT; ++i) af[i] = a[kr * K::LDA + i * 8];
#pragma unroll
      for (int j = 0; j < K::NT; ++j) bf[j] = b[kr * K::LDB + j * 8];
#pragma unroll
      for (int i = 0; i < K::MT; ++i)
#pragma unroll
        for (int j = 0; j < K::NT; ++j) dmma884(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: C = beta*C + alpha*acc (beta == 0: C not read), output permutation via strides
  const bool part = g.flags & kGroupPartial;
  double* Cb = (part ? p.P : p.C) + g.c_off;
  const double alpha = part ? 1.0 : p.alpha, beta = part ? 0.0 : p.beta;
#pragma unroll
  for (int i = 0; i < K::MT; ++i) {
    const int m = m0 + wm * K::WTM + i * 8 + fr_r;
    if (m >= M) continue;
    const int32_t om = dot_decode(m, nM, g.mext, g.cm_str);
#pragma unroll
    for (int j = 0; j < K::NT; ++j) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int n = n0 + wn * K::WTN + j * 8 + 2 * fr_k + r;
        if (n >= N) continue;
        double* c = Cb + om + dot_decode(n, nN, g.next, g.cn_str);
        const double v = __dmul_rn(alpha, acc[i][j][r]);
        *c = (beta == 0.0) ? v : __fma_rn(beta, *c, v);
      }
    }
  }
}

// Tile variants: chosen per plan to minimise padded work and wave quantisation.
using V0 = Cfg<128, 128, 16, 2, 4, 4, 1>;   // 8 warps, warp tile 64x32, 1 CTA/SM
using V1 = Cfg<80, 80, 16, 2, 2, 4, 2>;     // 4 warps, warp tile 40x40, 2 CTA/SM
using V2 = Cfg<64, 64, 16, 2, 2, 4, 3>;     // 4 warps, warp tile 32x32, 3 CTA/SM

int num_contract_variants() { return 3; }

VariantInfo contract_variant_info(int v) {
  switch (v) {
    case 0: return {V0::BM, V0::BN, V0::BK, V0::NTHREADS, V0::SMEM, 1, "128x128x16_w8"};
    case 1: return {V1::BM, V1::BN, V1::BK, V1::NTHREADS, V1::SMEM, 2, "80x80x16_w4"};
    default: return {V2::BM, V2::BN, V2::BK, V2::NTHREADS, V2::SMEM, 3, "64x64x16_w4"};
  }
}

template <class K, bool A, bool B>
static cudaError_t setup_one() {
  return cudaFuncSetAttribute(tt_contract_kernel<K, A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
}
template <class K>
static cudaError_t setup_cfg() {
  cudaError_t e;
  if ((e = setup_one<K, true, true>()) != cudaSuccess) return e;
  if ((e = setup_one<K, true, false>()) != cudaSuccess) return e;
  if ((e = setup_one<K, false, true>()) != cudaSuccess) return e;
  return setup_one<K, false, false>();
}

cudaError_t contract_variant_setup(int v) {
  switch (v) {
    case 0: return setup_cfg<V0>();
    case 1: return setup_cfg<V1>();
    default: return setup_cfg<V2>();
  }
}

template <class K>
static cudaError_t launch_cfg(bool akc, bool bnc, const ContractParams& p, int64_t nwork, cudaStream_t s) {
  dim3 grid((unsigned)nwork), block(K::NTHREADS);
  if (akc && bnc) tt_contract_kernel<K, true, true><<<grid, block, K::SMEM, s>>>(p);
  else if (akc) tt_contract_kernel<K, true, false><<<grid, block, K::SMEM, s>>>(p);
  else if (bnc) tt_contract_kernel<K, false, true><<<grid, block, K::SMEM, s>>>(p);
  else tt_contract_kernel<K, false, false><<<grid, block, K::SMEM, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_contract(int v, bool akc, bool bnc, const ContractParams& p, int64_t nwork, cudaStream_t s) {
  if (nwork <= 0) return cudaSuccess;
  switch (v) {
    case 0: return launch_cfg<V0>(akc, bnc, p, nwork, s);
    case 1: return launch_cfg<V1>(akc, bnc, p, nwork, s);
    default: return launch_cfg<V2>(akc, bnc, p, nwork, s);
  }
}

// ------------------------------------------------------------------------------------------------
// Device task-list builder: count -> scan -> fill (canonical order, reading R11)

__device__ __forceinline__ void tuple_blocks(const BuildParams& p, const int32_t* cc, int64_t t,
                                             int64_t& aid, int64_t& bid, int32_t* kc) {
  for (int l = p.nk - 1; l >= 0; --l) { kc[l] = (int32_t)(t % p.k_grid[l]); t /= p.k_grid[l]; }
  aid = 0;
  for (int d = 0; d < p.a_order; ++d) {
    int u = p.a_lab[d];
    aid = aid * p.a_grid[d] + (u < p.nc ? cc[u] : kc[u - p.nc]);
  }
  bid = 0;
  for (int d = 0; d < p.b_order; ++d) {
    int u = p.b_lab[d];
    bid = bid * p.b_grid[d] + (u < p.nc ? cc[u] : kc[u - p.nc]);
  }
}

__device__ __forceinline__ void cblock_coords(const BuildParams& p, int64_t cb, int32_t* cc) {
  for (int d = p.nc - 1; d >= 0; --d) { cc[d] = (int32_t)(cb % p.c_grid[d]); cb /= p.c_grid[d]; }
}

__global__ void build_count_kernel(const BuildParams p) {
  __shared__ int64_t red[32];
  int32_t cc[TT_MAX_ORDER], kc[TT_MAX_ORDER];
  cblock_coords(p, p.cblocks[blockIdx.x], cc);
  int64_t cnt = 0;
  for (int64_t t = threadIdx.x; t < p.ntuples; t += blockDim.x) {
    int64_t aid, bid;
    tuple_blocks(p, cc, t, aid, bid, kc);
    cnt += (p.a_nz[aid] && p.b_nz[bid]) ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    p.counts[blockIdx.x] = s;
  }
}

__global__ void build_scan_kernel(const BuildParams p) {
  // single CTA, 1024 threads, chunked exclusive scan of counts -> ptr
  __shared__ int64_t buf[1024];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < p.ncb; base += 1024) {
    int i = base + threadIdx.x;
    int64_t v = (i < p.ncb) ? p.counts[i] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      int64_t x = (threadIdx.x >= (unsigned)o) ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += x;
      __syncthreads();
    }
    if (i < p.ncb) p.ptr[i] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) p.ptr[p.ncb] = carry;
}

__global__ void build_fill_kernel(const BuildParams p) {
  __shared__ int32_t wsum[32];
  __shared__ int64_t base;
  int32_t cc[TT_MAX_ORDER], kc[TT_MAX_ORDER];
  cblock_coords(p, p.cblocks[blockIdx.x], cc);
  if (threadIdx.x == 0) base = p.ptr[blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t t0 = 0; t0 < p.ntuples; t0 += blockDim.x) {
    const int64_t t = t0 + threadIdx.x;
    int64_t aid = 0, bid = 0;
    bool f = false;
    if (t < p.ntuples) {
      tuple_blocks(p, cc, t, aid, bid, kc);
      f = p.a_nz[aid] && p.b_nz[bid];
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int64_t pos = base;
    for (int i = 0; i < warp; ++i) pos += wsum[i];
    pos += __popc(bal & ((1u << lane) - 1u));
    int64_t tot = 0;
    for (int i = 0; i < nw; ++i) tot += wsum[i];
    if (f) {
      p.a_blk[pos] = aid;
      p.b_blk[pos] = bid;
      // extents of every universal label in this task
      int32_t ext[kMaxLab];
      for (int u = 0; u < p.nc + p.nk; ++u) {
        const int tile = (u < p.nc) ? cc[u] : kc[u - p.nc];
        ext[u] = (int32_t)(p.lab_toff[u][tile + 1] - p.lab_toff[u][tile]);
      }
      int32_t sa[TT_MAX_ORDER], sb[TT_MAX_ORDER];
      int32_t acc = 1;
      for (int d = p.a_order - 1; d >= 0; --d) { sa[d] = acc; acc *= ext[p.a_lab[d]]; }
      acc = 1;
      for (int d = p.b_order - 1; d >= 0; --d) { sb[d] = acc; acc *= ext[p.b_lab[d]]; }
      TaskDesc td;
      td.a_off = p.a_boff[aid];
      td.b_off = p.b_boff[bid];
      td.pad = 0;
      int32_t K = 1;
      for (int gi = 0; gi < kMaxGroup; ++gi) {
        td.kext[gi] = 1; td.ak_str[gi] = 0; td.bk_str[gi] = 0; td.am_str[gi] = 0; td.bn_str[gi] = 0;
      }
      for (int gi = 0; gi < p.nK; ++gi) {
        int32_t e = 1;
        for (int q = 0; q < p.k_cnt[gi]; ++q) e *= ext[p.glab[p.k_first[gi] + q]];
        const int last = p.glab[p.k_first[gi] + p.k_cnt[gi] - 1];
        td.kext[gi] = e;
        td.ak_str[gi] = sa[p.a_pos[last]];
        td.bk_str[gi] = sb[p.b_pos[last]];
        K *= e;
      }
      for (int gi = 0; gi < p.nM; ++gi) td.am_str[gi] = sa[p.a_pos[p.glab[p.m_first[gi] + p.m_cnt[gi] - 1]]];
      for (int gi = 0; gi < p.nN; ++gi) td.bn_str[gi] = sb[p.b_pos[p.glab[p.n_first[gi] + p.n_cnt[gi] - 1]]];
      td.K = K;
      p.tasks[pos] = td;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
}

cudaError_t launch_build_count(const BuildParams& p, cudaStream_t s) {
  if (p.ncb <= 0) return cudaSuccess;
  build_count_kernel<<<p.ncb, 256, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_build_scan(const BuildParams& p, cudaStream_t s) {
  build_scan_kernel<<<1, 1024, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_build_fill(const BuildParams& p, cudaStream_t s) {
  if (p.ncb <= 0) return cudaSuccess;
  build_fill_kernel<<<p.ncb, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// Element kernels.  One CTA per segment (a contiguous element range of one block), or per 32x32
// tile in transpose mode.  HBM-bound: vectorised contiguous paths, multiply-high index decode.

constexpr int kElemThreads = 256;

// all threads of the CTA copy a descriptor into shared memory (word-parallel), then barrier
template <class T>
__device__ __forceinline__ void load_desc(T& dst, const T* src) {
  static_assert(sizeof(T) % 4 == 0, "descriptor size");
  const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
  uint32_t* d = reinterpret_cast<uint32_t*>(&dst);
  const int tid = threadIdx.x + threadIdx.y * blockDim.x, nt = blockDim.x * blockDim.y;
  for (int i = tid; i < (int)(sizeof(T) / 4); i += nt) d[i] = s[i];
  __syncthreads();
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  const uint32_t t = __umulhi(n, f.m);
  return (t + n) >> f.l;
}

// x-order element index (row-major over the groups) -> offset in the other operand
__device__ __forceinline__ int64_t y_offset(uint32_t e, const ElemDesc& d) {
  int64_t off = 0;
  for (int g = d.n - 1; g > 0; --g) {
    const uint32_t q = fdiv(e, d.div[g]);
    off += (int64_t)(e - q * d.div[g].d) * d.y_str[g];
    e = q;
  }
  return off + (int64_t)e * d.y_str[0];
}

__global__ void set_kernel(const ElemParams p) {
  const Segment sg = p.segs[blockIdx.x];
  double* x = p.X + p.descs[sg.desc].x_off;
  // blocks are 16-B aligned: peel an odd first element, double2 stores, scalar tail
  const int64_t es = sg.e0 + (sg.e0 & 1);
  const int64_t n2 = (sg.e1 - es) / 2;
  double2* x2 = reinterpret_cast<double2*>(x + es);
  const double2 v = make_double2(p.alpha, p.alpha);
  for (int64_t i = threadIdx.x; i < n2; i += blockDim.x) x2[i] = v;
  if (threadIdx.x == 0 && es != sg.e0 && sg.e0 < sg.e1) x[sg.e0] = p.alpha;
  if (threadIdx.x == 0 && es + 2 * n2 < sg.e1) x[sg.e1 - 1] = p.alpha;
}

// row index over the groups 0..n-2 (rows mode: group n-1 is contiguous in y) -> offset in y
__device__ __forceinline__ int64_t y_row_offset(uint32_t r, const ElemDesc& d) {
  int64_t off = 0;
  for (int g = d.n - 2; g > 0; --g) {
    const uint32_t q = fdiv(r, d.div[g]);
    off += (int64_t)(r - q * d.div[g].d) * d.y_str[g];
    r = q;
  }
  return off + (int64_t)r * d.y_str[0];
}

// rows mode walks 16-B pairs: needs an even row length, even Y strides and even block offsets (else the
// generic per-element decode runs)
__device__ __forceinline__ bool rows_pairs(const ElemDesc& d) {
  bool ok = (d.div[d.n - 1].d % 2 == 0) && (d.x_off % 2 == 0) && (d.y_off < 0 || d.y_off % 2 == 0);
  for (int g = 0; g < d.n - 1; ++g) ok = ok && (d.y_str[g] % 2 == 0);
  return ok;
}

// beta*x + alpha*y with ONE rounding order in every kernel and block mode (explicit intrinsics: the
// compiler never re-associates or contracts them differently per call site), so that a block gives the
// same bits whether it runs as tiles, rows or segments (e.g. whole vs row-split blocks, R12)
__device__ __forceinline__ double axpby(double alpha, double y, double beta, double x) {
  const double t = __dmul_rn(alpha, y);
  return (beta == 0.0) ? t : __fma_rn(beta, x, t);
}

// Deterministic warp-then-CTA sum of one value per thread (fixed shuffle tree, warps in order).
__device__ __forceinline__ double cta_sum(double s, double* warp_sums) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  const int tid = threadIdx.x + threadIdx.y * blockDim.x, nw = (blockDim.x * blockDim.y) / 32;
  if ((tid & 31) == 0) warp_sums[tid >> 5] = s;
  __syncthreads();
  double t = 0.0;
  if (tid == 0)
    for (int w = 0; w < nw; ++w) t += warp_sums[w];
  return t;
}

constexpr int kElemUnroll = 4;   // elements per thread in flight (generic decode path)

// Segment work (descriptors in contiguous or generic mode; the mode is per descriptor, uniform per
// CTA).  Every thread issues all its loads of a batch before any store (X and Y are distinct
// buffers: __restrict__), so each thread keeps kElemUnroll loads of each operand in flight.
__global__ void __launch_bounds__(kElemThreads) add_seg_kernel(const ElemParams p) {
  __shared__ ElemDesc d;
  const Segment sg = p.segs[blockIdx.x];
  load_desc(d, p.descs + sg.desc);
  double* __restrict__ x = p.X + d.x_off;
  const double* __restrict__ y = (d.y_off >= 0) ? p.Y + d.y_off : nullptr;
  const double alpha = p.alpha, beta = p.beta;
  if (d.mode == kElemContig) {
    const int64_t es = sg.e0 + (sg.e0 & 1);
    const int64_t n2 = (sg.e1 - es) / 2;
    double2* __restrict__ x2 = reinterpret_cast<double2*>(x + es);
    const double2* __restrict__ y2 = y ? reinterpret_cast<const double2*>(y + es) : nullptr;
    for (int64_t i0 = threadIdx.x; i0 < n2; i0 += kElemThreads * 2) {
      double2 v[2], o[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t i = i0 + u * kElemThreads;
        v[u] = (y2 && i < n2) ? y2[i] : make_double2(0.0, 0.0);
        o[u] = (beta != 0.0 && i < n2) ? x2[i] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t i = i0 + u * kElemThreads;
        if (i < n2) x2[i] = make_double2(axpby(alpha, v[u].x, beta, o[u].x), axpby(alpha, v[u].y, beta, o[u].y));
      }
    }
    if (threadIdx.x == 0) {
      int64_t peel[2] = {es != sg.e0 ? sg.e0 : -1, es + 2 * n2 < sg.e1 ? sg.e1 - 1 : -1};
      for (int64_t e : peel) {
        if (e < 0) continue;
        x[e] = axpby(alpha, y ? y[e] : 0.0, beta, beta != 0.0 ? x[e] : 0.0);
      }
    }
  } else if (d.mode == kElemRows && rows_pairs(d)) {
    // rows of L elements contiguous in both operands, walked flat: consecutive threads take consecutive
    // 16-B pairs of X (fully coalesced), each decoding its row's Y base (Y read in runs of L)
    const uint32_t L = d.div[d.n - 1].d;
    const int64_t es = sg.e0 + (sg.e0 & 1);
    const int64_t n2 = (sg.e1 - es) / 2;
    double2* __restrict__ x2 = reinterpret_cast<double2*>(x + es);
    for (int64_t i0 = threadIdx.x; i0 < n2; i0 += kElemThreads * kElemUnroll) {
      double2 v[kElemUnroll], o[kElemUnroll];
#pragma unroll
      for (int u = 0; u < kElemUnroll; ++u) {
        const int64_t i = i0 + u * kElemThreads;
        v[u] = o[u] = make_double2(0.0, 0.0);
        if (i < n2) {
          const uint32_t e = (uint32_t)(es + 2 * i), r = fdiv(e, d.div[d.n - 1]);
          if (y) v[u] = *reinterpret_cast<const double2*>(y + y_row_offset(r, d) + (e - r * L));
          if (beta != 0.0) o[u] = x2[i];
        }
      }
#pragma unroll
      for (int u = 0; u < kElemUnroll; ++u) {
        const int64_t i = i0 + u * kElemThreads;
        if (i < n2) x2[i] = make_double2(axpby(alpha, v[u].x, beta, o[u].x), axpby(alpha, v[u].y, beta, o[u].y));
      }
    }
    if (threadIdx.x == 0) {
      int64_t peel[2] = {es != sg.e0 ? sg.e0 : -1, es + 2 * n2 < sg.e1 ? sg.e1 - 1 : -1};
      for (int64_t e : peel) {
        if (e < 0) continue;
        x[e] = axpby(alpha, y ? y[y_offset((uint32_t)e, d)] : 0.0, beta, beta != 0.0 ? x[e] : 0.0);
      }
    }
  } else {
    for (int64_t e0 = sg.e0 + threadIdx.x; e0 < sg.e1; e0 += kElemThreads * kElemUnroll) {
      double yv[kElemUnroll], xv[kElemUnroll];
#pragma unroll
      for (int u = 0; u < kElemUnroll; ++u) {
        const int64_t e = e0 + u * kElemThreads;
        yv[u] = (y && e < sg.e1) ? y[y_offset((uint32_t)e, d)] : 0.0;
        xv[u] = (beta != 0.0 && e < sg.e1) ? x[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kElemUnroll; ++u) {
        const int64_t e = e0 + u * kElemThreads;
        if (e < sg.e1) x[e] = axpby(alpha, yv[u], beta, xv[u]);
      }
    }
  }
}

// Transpose work: one 32x32 tile per CTA (32 x 8 threads, 4 elements each).  Bases and strides come
// precomputed in the TileItem (no descriptor decode).  All loads -- Y along its contiguous group into
// registers, and (beta != 0) X along its contiguous group -- are issued before the barrier; Y goes
// through a padded shared tile so both the reads and the writes are 256-B coalesced rows.
__global__ void __launch_bounds__(256) add_tile_kernel(const ElemParams p) {
  __shared__ double tile[32][33];
  const TileItem t = p.tiles[blockIdx.x];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const double* __restrict__ y = p.Y;
  double* __restrict__ x = p.X;
  const double alpha = p.alpha, beta = p.beta;
  double yv[4], xv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {   // read: lanes along the y-contiguous group (iy), rows along ix
    const int ix = ly + 8 * k, iy = lx;
    yv[k] = (t.y_base >= 0 && ix < t.nx && iy < t.ny) ? y[t.y_base + (int64_t)ix * t.y_ld + iy] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {   // write side: lanes along ix (x contiguous), rows along iy
    const int ix = lx, iy = ly + 8 * k;
    xv[k] = (beta != 0.0 && ix < t.nx && iy < t.ny) ? x[t.x_base + (int64_t)iy * t.x_ld + ix] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) tile[ly + 8 * k][lx] = yv[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ix = lx, iy = ly + 8 * k;
    if (ix < t.nx && iy < t.ny) x[t.x_base + (int64_t)iy * t.x_ld + ix] = axpby(alpha, tile[ix][iy], beta, xv[k]);
  }
}

// Scalar partial of one 32x32 tile (one per CTA; fixed order: per thread, shuffle tree, warps in order).
__global__ void __launch_bounds__(256) scalar_tile_kernel(const ElemParams p, double* __restrict__ partials) {
  __shared__ double tile[32][33];
  __shared__ double wsum[8];
  const TileItem t = p.tiles[blockIdx.x];
  const int lx = threadIdx.x, ly = threadIdx.y;
  const double* __restrict__ y = p.Y;
  const double* __restrict__ x = p.X;
  double yv[4], xv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ix = ly + 8 * k, iy = lx;
    yv[k] = (ix < t.nx && iy < t.ny) ? y[t.y_base + (int64_t)ix * t.y_ld + iy] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ix = lx, iy = ly + 8 * k;
    xv[k] = (ix < t.nx && iy < t.ny) ? x[t.x_base + (int64_t)iy * t.x_ld + ix] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) tile[ly + 8 * k][lx] = yv[k];
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += xv[k] * tile[lx][ly + 8 * k];
  s = cta_sum(s, wsum);
  if (lx == 0 && ly == 0) partials[blockIdx.x] = s;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_kernel(const ElemParams p) {
  const Segment sg = p.segs[blockIdx.x];
  const ElemDesc d = p.descs[sg.desc];
  double* x = p.X + d.x_off;
  for (int64_t e = sg.e0 + threadIdx.x; e < sg.e1; e += blockDim.x) {
    uint32_t r = (uint32_t)e;
    int64_t g = d.g_origin;
    for (int q = p.order - 1; q > 0; --q) {
      const uint32_t qq = fdiv(r, d.div[q]);
      g += (int64_t)(r - qq * d.div[q].d) * d.g_str[q];
      r = qq;
    }
    g += (int64_t)r * d.g_str[0];
    const uint64_t h = splitmix64(p.key ^ (uint64_t)g);
    x[e] = (p.kind == TT_KIND_INTEGER) ? (double)(int64_t)(h % 5ull) - 2.0
                                       : (double)(h >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
  }
}

// Deterministic: each CTA sums its segment in a fixed order (per thread, shuffle tree, warps in order).
__global__ void __launch_bounds__(kElemThreads) scalar_seg_kernel(const ElemParams p) {
  __shared__ double wsum[kElemThreads / 32];
  __shared__ ElemDesc d;
  const Segment sg = p.segs[blockIdx.x];
  load_desc(d, p.descs + sg.desc);
  const double* __restrict__ x = p.X + d.x_off;
  const double* __restrict__ y = p.Y + d.y_off;
  double s = 0.0;
  if (d.mode == kElemContig) {
    const int64_t es = sg.e0 + (sg.e0 & 1);
    const int64_t n2 = (sg.e1 - es) / 2;
    const double2* __restrict__ x2 = reinterpret_cast<const double2*>(x + es);
    const double2* __restrict__ y2 = reinterpret_cast<const double2*>(y + es);
    for (int64_t i0 = threadIdx.x; i0 < n2; i0 += kElemThreads * 2) {
      double2 a[2], b[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t i = i0 + u * kElemThreads;
        a[u] = i < n2 ? x2[i] : make_double2(0.0, 0.0);
        b[u] = i < n2 ? y2[i] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        s += a[u].x * b[u].x;
        s += a[u].y * b[u].y;
      }
    }
    if (threadIdx.x == 0 && es != sg.e0 && sg.e0 < sg.e1) s += x[sg.e0] * y[sg.e0];
    if (threadIdx.x == 0 && es + 2 * n2 < sg.e1) s += x[sg.e1 - 1] * y[sg.e1 - 1];
  } else if (d.mode == kElemRows && rows_pairs(d)) {
    // as in add_seg_kernel: flat 16-B pairs of X, the row's Y base decoded per pair
    const uint32_t L = d.div[d.n - 1].d;
    const int64_t es = sg.e0 + (sg.e0 & 1);
    const int64_t n2 = (sg.e1 - es) / 2;
    const double2* __restrict__ x2 = reinterpret_cast<const double2*>(x + es);
    for (int64_t i0 = threadIdx.x; i0 < n2; i0 += kElemThreads * kElemUnroll) {
      double2 a[kElemUnroll], b[kElemUnroll];
#pragma unroll
      for (int u = 0; u < kElemUnroll; ++u) {
        const int64_t i = i0 + u * kElemThreads;
        a[u] = b[u] = make_double2(0.0, 0.0);
        if (i < n2) {
          const uint32_t e = (uint32_t)(es + 2 * i), r = fdiv(e, d.div[d.n - 1]);
          a[u] = x2[i];
          b[u] = *reinterpret_cast<const double2*>(y + y_row_offset(r, d) + (e - r * L));
        }
      }
#pragma unroll
      for (int u = 0; u < kElemUnroll; ++u) {
        s += a[u].x * b[u].x;
        s += a[u].y * b[u].y;
      }
    }
    if (threadIdx.x == 0 && es != sg.e0 && sg.e0 < sg.e1) s += x[sg.e0] * y[y_offset((uint32_t)sg.e0, d)];
    if (threadIdx.x == 0 && es + 2 * n2 < sg.e1) s += x[sg.e1 - 1] * y[y_offset((uint32_t)(sg.e1 - 1), d)];
  } else {
    for (int64_t e0 = sg.e0 + threadIdx.x; e0 < sg.e1; e0 += kElemThreads * kElemUnroll) {
      double yv[kElemUnroll], xv[kElemUnroll];
#pragma unroll
      for (int u = 0; u < kElemUnroll; ++u) {
        const int64_t e = e0 + u * kElemThreads;
        yv[u] = e < sg.e1 ? y[y_offset((uint32_t)e, d)] : 0.0;
        xv[u] = e < sg.e1 ? x[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kElemUnroll; ++u) s += xv[u] * yv[u];
    }
  }
  s = cta_sum(s, wsum);
  if (threadIdx.x == 0) p.partials[blockIdx.x] = s;
}

// First stage of the final sum when there are many partials: CTA c sums partials [c*4096, (c+1)*4096)
// in a fixed order.
constexpr int kFinalChunk = 4096;
__global__ void __launch_bounds__(256) scalar_stage_kernel(const double* __restrict__ partials, int64_t n,
                                                           double* __restrict__ out) {
  __shared__ double wsum[8];
  const int64_t b = (int64_t)blockIdx.x * kFinalChunk, e = min(n, b + kFinalChunk);
  double s = 0.0;
  for (int64_t i = b + threadIdx.x; i < e; i += 256) s += partials[i];
  s = cta_sum(s, wsum);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void scalar_final_kernel(const double* partials, int64_t n, double alpha, double* out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = alpha * red[0];
}

cudaError_t launch_set(const ElemParams& p, int64_t nseg, cudaStream_t s) {
  if (nseg <= 0) return cudaSuccess;
  set_kernel<<<(unsigned)nseg, kElemThreads, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_add(const ElemParams& p, int64_t nseg, int64_t ntiles, cudaStream_t s) {
  if (nseg > 0) add_seg_kernel<<<(unsigned)nseg, kElemThreads, 0, s>>>(p);
  if (ntiles > 0) add_tile_kernel<<<(unsigned)ntiles, dim3(32, 8), 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_fill(const ElemParams& p, int64_t nseg, cudaStream_t s) {
  if (nseg <= 0) return cudaSuccess;
  fill_kernel<<<(unsigned)nseg, kElemThreads, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_scalar_partials(const ElemParams& p, int64_t nseg, int64_t ntiles, cudaStream_t s) {
  if (nseg > 0) scalar_seg_kernel<<<(unsigned)nseg, kElemThreads, 0, s>>>(p);
  if (ntiles > 0) scalar_tile_kernel<<<(unsigned)ntiles, dim3(32, 8), 0, s>>>(p, p.partials + nseg);
  return cudaGetLastError();
}
int64_t scalar_scratch_elems(int64_t n) { return n > kFinalChunk ? (n + kFinalChunk - 1) / kFinalChunk : 0; }

// simulated-rank all-reduce: out = part[0] + part[1] + ... in rank order
__global__ void sum_slots_kernel(const double* __restrict__ part, int32_t n, double* __restrict__ out) {
  double s = 0.0;
  for (int32_t i = 0; i < n; ++i) s += part[i];
  *out = s;
}
cudaError_t launch_sum_slots(const double* part, int32_t n, double* out, cudaStream_t s) {
  sum_slots_kernel<<<1, 1, 0, s>>>(part, n, out);
  return cudaGetLastError();
}

cudaError_t launch_scalar_final(const double* partials, int64_t n, double alpha, double* out, double* scratch,
                               cudaStream_t s) {
  const int64_t n1 = scratch ? scalar_scratch_elems(n) : 0;
  if (n1 > 0) {
    scalar_stage_kernel<<<(unsigned)n1, 256, 0, s>>>(partials, n, scratch);
    scalar_final_kernel<<<1, 1024, 0, s>>>(scratch, n1, alpha, out);
  } else {
    scalar_final_kernel<<<1, 1024, 0, s>>>(partials, n, alpha, out);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// Split-K reduction (contractions with too few output tiles to fill the GPU): the chunks of a C part
// wrote raw sums into slots of P laid out like the C block; C = beta*C + alpha * (slot 0 + slot 1 + ...)
// in slot order -- deterministic (R12).  blockIdx.y = split descriptor; threads stride its elements.
__global__ void split_reduce_kernel(const double* __restrict__ P, double* __restrict__ C,
                                    const CGroupDesc* __restrict__ groups, const SplitDesc* __restrict__ splits,
                                    int32_t nM, int32_t nN, double alpha, double beta) {
  const SplitDesc sd = splits[blockIdx.y];
  const CGroupDesc& g = groups[sd.group];
  const int32_t rows = g.M - g.m_begin, cols = g.N - g.n_begin;
  const int64_t n = (int64_t)rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t m = g.m_begin + (int32_t)(e / cols), c = g.n_begin + (int32_t)(e % cols);
    const int64_t off = dot_decode(m, nM, g.mext, g.cm_str) + dot_decode(c, nN, g.next, g.cn_str);
    const double* ps = P + sd.p_off + off;
    double acc = 0.0;
    for (int32_t s = 0; s < sd.nslots; ++s) acc += ps[(int64_t)s * sd.vol];
    double* o = C + sd.c_off + off;
    const double v = __dmul_rn(alpha, acc);
    *o = (beta == 0.0) ? v : __fma_rn(beta, *o, v);
  }
}

cudaError_t launch_split_reduce(const double* P, double* C, const CGroupDesc* groups, const SplitDesc* splits,
                                int32_t nsplit, int32_t nM, int32_t nN, double alpha, double beta, cudaStream_t s) {
  if (nsplit <= 0) return cudaSuccess;
  split_reduce_kernel<<<dim3(16, (unsigned)nsplit), 256, 0, s>>>(P, C, groups, splits, nM, nN, alpha, beta);
  return cudaGetLastError();
}

}  // namespace tt
