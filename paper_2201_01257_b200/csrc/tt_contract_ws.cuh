// tt_contract_ws.cuh -- warp-specialised block-sparse FP64 contraction kernel for sm_100a.
//
// Same work decomposition and descriptors as tt_contract_kernel (tt_kernels.cu), reorganised for
// Blackwell's asynchronous pipeline style:
//   * PRODUCER warps (one per operand) stream the A and B tiles of every (task, BK slice) straight
//     from their native block layout into a STAGES-deep shared-memory ring with cp.async (16-byte
//     copies along the operand's contiguous direction when its innermost extent is even), and
//     signal a per-stage "full" mbarrier with cp.async.mbarrier.arrive.noinc.  The index
//     permutation of each operand (TAMM's HPTT/LibreTT pass, P107/P220) is folded into these source
//     addresses via the label-group strides of the task descriptor.
//   * MMA warps wait on "full", load fragments and issue FP64 tensor-core MMAs (mma.sync m8n8k4 ->
//     DMMA.8x8x4), then release the slot on an "empty" mbarrier.  No CTA-wide barrier in the loop.
//   * Shared-memory layouts are chosen so that both the cp.async writes and the fragment loads are
//     bank-conflict free: the contiguous direction of the operand stays contiguous in smem;
//     k-contiguous tiles use rows of BK+8 doubles (row stride = 64 mod 128 B, fragment loads are
//     128-bit and cover two DMMA k-steps), row-contiguous tiles use rows of R+2 doubles (row stride
//     = 16 mod 64 B, the two k-steps of an 8-wide k octet use k = 2*(lane%4) + t).
//   * Accumulation over all pairs of an output tile stays in registers in canonical task order
//     (deterministic, reading R12); epilogue C = beta*C + alpha*acc through the C strides.
#pragma once
#include <cstdint>

#include <cuda.h>

#include "tt_launch.h"

namespace tt {

namespace ws {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(s));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(s) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(s),
      "r"(parity)
      : "memory");
}
// producer-side wait: back off so that idle producers do not take issue slots from the MMA warps
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  unsigned ok = 0;
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(s), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(64);
  }
}
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

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

// Shared-memory geometry of one operand tile (R rows = BM or BN, BK k's).
template <int R, int BK, bool KC>
struct Tile {
  static constexpr int LD = KC ? (BK + 8) : (R + 2);     // doubles per smem row
  static constexpr int ELEMS = KC ? R * LD : BK * LD;     // doubles per stage
};

// Copy geometry of one operand for one producer warp.
//   KC (k contiguous in global and smem):  lane -> (row = lane / 8, k unit = lane % 8); a k unit is
//       a 16-B pair (VEC) or, without VEC, two single doubles k and k+8.  NR = R/4 rows per lane.
//   !KC (rows contiguous): lane -> (row unit = lane % QL, k = lane / QL + (32/QL)*j); a row unit is
//       a 16-B pair (VEC) or a single double.  NR row units per lane, NK k values per lane.
template <int R, int BK, bool KC, bool VEC>
struct Copy {
  static constexpr int RU = VEC ? 2 : 1;                            // rows per unit (row-contig)
  static constexpr int QL = KC ? 8 : ((R / RU) % 32 == 0 ? 32 : ((R / RU) % 16 == 0 ? 16 : 8));
  static constexpr int NR = KC ? R / 4 : (R / RU) / QL;
  static constexpr int NK = KC ? (VEC ? 1 : 2) : BK / (32 / QL);
  static_assert(KC ? (R % 4 == 0) : ((R / RU) % QL == 0), "copy geometry");
  static_assert(KC || (BK % (32 / QL) == 0), "copy geometry k");
};

template <int BM_, int BN_, int BK_, int WM_, int WN_, int MAXSTAGES_, int MINB_>
struct WCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, MAXSTAGES = MAXSTAGES_, MINB = MINB_;
  static constexpr int NMMA = WM * WN, NPROD = 2, NW = NMMA + NPROD, NTHREADS = NW * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN, MT = WTM / 8, NT = WTN / 8;
  static_assert(BK % 8 == 0, "BK multiple of 8 (k octets)");
};

template <class K, bool AKC, bool BNC>
struct Smem {
  static constexpr bool BKC = !BNC;
  using TA = Tile<K::BM, K::BK, AKC>;
  using TB = Tile<K::BN, K::BK, BKC>;
  static constexpr int A_ELEMS = TA::ELEMS, B_ELEMS = TB::ELEMS;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  // as many stages as fit the shared-memory budget of MINB CTAs per SM (227 KB per SM usable)
  static constexpr int BUDGET = (227 * 1024) / K::MINB - 1024;
  static constexpr int FIT = BUDGET / (STAGE * 8 + 16);
  static constexpr int STAGES = FIT < K::MAXSTAGES ? FIT : K::MAXSTAGES;
  static constexpr int BYTES = STAGES * STAGE * 8 + 2 * STAGES * 8 + 256;
  static_assert(STAGES >= 3, "pipeline too shallow");
};

// Producer: stream one operand for every work item of this (persistent) CTA.  ROWS = BM (A) or BN
// (B); KC = k contiguous.  The stage ring and its phases continue across work items, so the next
// item's first stages are in flight while the MMA warps finish the current item and its epilogue.
template <class K, int STAGES, int ROWS, bool KC, bool VEC>
__device__ __forceinline__ void produce(const ContractParams& p, bool isA, double* sbase, int stage_elems, int ld,
                                        uint64_t* full, uint64_t* empty) {
  using C = Copy<ROWS, K::BK, KC, VEC>;
  const int lane = threadIdx.x & 31;
  const int nG = isA ? p.nM : p.nN;                 // row groups
  const int nK = p.nK;
  // lane geometry
  const int r_l = KC ? (lane >> 3) : (lane % C::QL) * C::RU;   // first row of the lane
  const int k_l = KC ? (lane & 7) * (VEC ? 2 : 1) : (lane / C::QL);
  const int r_step = KC ? 4 : C::QL * C::RU;
  const int k_step = KC ? 8 : 32 / C::QL;          // (!VEC KC: second k at +8)
  int32_t roff[C::NR];
  int32_t kext[kMaxGroup], kst[kMaxGroup], rext[kMaxGroup];
  const double* base = nullptr;
  int32_t Kt = 0;
  int st = 0;
  unsigned phase = 1;   // empty barriers: first wait passes
  for (int64_t wi = blockIdx.x; wi < p.nwork; wi += gridDim.x) {
    const WorkItem w = p.work[wi];
    const CGroupDesc* g = p.groups + w.group;
    const int row0 = isA ? g->m_begin + w.mt * K::BM : g->n_begin + w.nt * K::BN;
    const int ROWMAX = isA ? g->M : g->N;
    const int t_end = g->task_end, nst = g->nstages;
#pragma unroll
    for (int i = 0; i < kMaxGroup; ++i) rext[i] = isA ? g->mext[i] : g->next[i];
    int t = g->task_begin, k0 = 0;
    auto setup = [&](int tt_) {
      const TaskDesc* td = p.tasks + tt_;
      base = isA ? p.A + td->a_off : p.B + td->b_off;
      Kt = td->K;
      int32_t rst[kMaxGroup];
#pragma unroll
      for (int i = 0; i < kMaxGroup; ++i) {
        kext[i] = td->kext[i];
        kst[i] = isA ? td->ak_str[i] : td->bk_str[i];
        rst[i] = isA ? td->am_str[i] : td->bn_str[i];
      }
#pragma unroll
      for (int i = 0; i < C::NR; ++i) {
        const int r = row0 + r_l + r_step * i;
        roff[i] = (r < ROWMAX) ? dot_decode(r, nG, rext, rst) : -1;
      }
    };
    if (t < t_end) setup(t);
    for (int s = 0; s < nst; ++s) {
      mbar_wait_sleep(&empty[st], phase);
      double* dst = sbase + st * stage_elems;
#pragma unroll
      for (int j = 0; j < C::NK; ++j) {
        const int kl = k_l + k_step * j;
        const int k = k0 + kl;
        const bool kv = k < Kt;
        const int32_t ko = kv ? dot_decode(k, nK, kext, kst) : 0;
#pragma unroll
        for (int i = 0; i < C::NR; ++i) {
          const int rl = r_l + r_step * i;
          const bool v = kv && roff[i] >= 0;
          const double* src = v ? base + roff[i] + ko : p.A;
          double* d = KC ? dst + rl * ld + kl : dst + kl * ld + rl;
          if (VEC) cp_async16(d, src, v);
          else cp_async8(d, src, v);
        }
      }
      mbar_arrive_cp_async(&full[st]);
      k0 += K::BK;
      if (k0 >= Kt) {
        k0 = 0;
        ++t;
        if (t < t_end) setup(t);
      }
      if (++st == STAGES) { st = 0; phase ^= 1; }
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Persistent CTAs (grid = min(work items, resident CTAs)): CTA b processes items b, b+G, b+2G, ...
// (items are sorted by cost, so striding balances like LPT).
template <class K, bool AKC, bool BNC, bool AVEC, bool BVEC>
__global__ void __launch_bounds__(K::NTHREADS, K::MINB) tt_contract_ws_kernel(const ContractParams p) {
  using SM = Smem<K, AKC, BNC>;
  constexpr bool BKC = !BNC;
  extern __shared__ __align__(128) double smem[];
  double* sA = smem;
  constexpr int STAGES = SM::STAGES;
  double* sB = smem + STAGES * SM::A_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SM::STAGE);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2 * 32);        // every producer thread arrives once per stage
      mbar_init(&empty[s], K::NMMA);      // one arrival per MMA warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= K::NMMA) {
    // ------------------------------------------------------------- producers
    if (warp == K::NMMA)
      produce<K, STAGES, K::BM, AKC, AVEC>(p, true, sA, SM::A_ELEMS, SM::TA::LD, full, empty);
    else
      produce<K, STAGES, K::BN, BKC, BVEC>(p, false, sB, SM::B_ELEMS, SM::TB::LD, full, empty);
    return;
  }

  // --------------------------------------------------------------- MMA warps
  const int wm = warp / K::WN, wn = warp % K::WN;
  const int q = lane & 3, r8 = lane >> 2;
  const double alpha_ = p.alpha, beta_ = p.beta;
  int st = 0;
  unsigned phase = 0;
  for (int64_t wi = blockIdx.x; wi < p.nwork; wi += gridDim.x) {
    const WorkItem w = p.work[wi];
    const CGroupDesc* g = p.groups + w.group;
    const int m0 = g->m_begin + w.mt * K::BM, n0 = g->n_begin + w.nt * K::BN;
    const int nst = g->nstages;
    double acc[K::MT][K::NT][2];
#pragma unroll
    for (int i = 0; i < K::MT; ++i)
#pragma unroll
      for (int j = 0; j < K::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int s = 0; s < nst; ++s) {
      mbar_wait(&full[st], phase);
      const double* a = sA + st * SM::A_ELEMS;
      const double* b = sB + st * SM::B_ELEMS;
#pragma unroll
      for (int o = 0; o < K::BK / 8; ++o) {
        double af[K::MT][2], bf[K::NT][2];
#pragma unroll
        for (int i = 0; i < K::MT; ++i) {
          const int m = wm * K::WTM + i * 8 + r8;
          if (AKC) {
            const double2 v = *reinterpret_cast<const double2*>(a + m * SM::TA::LD + 8 * o + 2 * q);
            af[i][0] = v.x;
            af[i][1] = v.y;
          } else {
            af[i][0] = a[(8 * o + 2 * q) * SM::TA::LD + m];
            af[i][1] = a[(8 * o + 2 * q + 1) * SM::TA::LD + m];
          }
        }
#pragma unroll
        for (int j = 0; j < K::NT; ++j) {
          const int n = wn * K::WTN + j * 8 + r8;
          if (BKC) {
            const double2 v = *reinterpret_cast<const double2*>(b + n * SM::TB::LD + 8 * o + 2 * q);
            bf[j][0] = v.x;
            bf[j][1] = v.y;
          } else {
            bf[j][0] = b[(8 * o + 2 * q) * SM::TB::LD + n];
            bf[j][1] = b[(8 * o + 2 * q + 1) * SM::TB::LD + n];
          }
        }
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int i = 0; i < K::MT; ++i)
#pragma unroll
            for (int j = 0; j < K::NT; ++j) dmma884(acc[i][j], af[i][t], bf[j][t]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == STAGES) { st = 0; phase ^= 1; }
    }

    // epilogue (the producers are already streaming the next item)
    const bool part = g->flags & kGroupPartial;
    double* Cb = (part ? p.P : p.C) + g->c_off;
    const double alpha = part ? 1.0 : alpha_, beta = part ? 0.0 : beta_;
    const int M = g->M, N = g->N;
    int32_t mext[kMaxGroup], next[kMaxGroup], cms[kMaxGroup], cns[kMaxGroup];
#pragma unroll
    for (int i = 0; i < kMaxGroup; ++i) {
      mext[i] = g->mext[i];
      next[i] = g->next[i];
      cms[i] = g->cm_str[i];
      cns[i] = g->cn_str[i];
    }
#pragma unroll
    for (int i = 0; i < K::MT; ++i) {
      const int m = m0 + wm * K::WTM + i * 8 + r8;
      if (m >= M) continue;
      const int32_t om = dot_decode(m, p.nM, mext, cms);
#pragma unroll
      for (int j = 0; j < K::NT; ++j) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int n = n0 + wn * K::WTN + j * 8 + 2 * q + r;
          if (n >= N) continue;
          double* c = Cb + om + dot_decode(n, p.nN, next, cns);
          const double v = __dmul_rn(alpha, acc[i][j][r]);
          *c = (beta == 0.0) ? v : __fma_rn(beta, *c, v);
        }
      }
    }
  }
}


// =================================================================================================
// TMA variant (fused GEMM-shaped operands with uniform blocks: the ladder / hole-hole layouts).
// One producer THREAD issues two 2-D cp.async.bulk.tensor loads per stage (A box {16 k, BM rows}
// with 128-byte swizzle, B box {BN+2 n, 16 k} unswizzled) that complete_tx on the stage's mbarrier;
// the tensor maps view the whole packed A / B buffer as [rows][K] / [rows][N] matrices (blocks of
// one shape are contiguous in packed order).  A rows beyond a block's M read the next block (their
// outputs are discarded), columns beyond K / N read zeros (TMA out-of-bounds fill).  A fragments read
// swizzled 16-byte chunks; the 8 rows of a fragment are permuted (r -> (r>>1) | ((r&1)<<2)) so that
// the two rows of every quarter-warp hit opposite 64-byte halves: conflict-free LDS.128.

__device__ __forceinline__ int perm8(int r) { return (r >> 1) | ((r & 1) << 2); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(s),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(d),
      "l"(map), "r"(x), "r"(y), "r"(b)
      : "memory");
}

// BKC: B is [N][K] in its blocks (k contiguous, e.g. the implicit operand's X(q,s,L)): its box is
// {16 k, BN rows} with the 128-byte swizzle of A and its fragments are read like A's.
__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(b)
      : "memory");
}

template <class K, bool BKC = false>
struct TmaSmem {
  static constexpr int A_BYTES = K::BM * 128;                 // BK = 16 doubles = 128 B rows, swizzled
  static constexpr int B_LD = K::BN + 2;                      // doubles per B row (box width; [K][N] B)
  static constexpr int B_BYTES = BKC ? K::BN * 128 : K::BK * B_LD * 8;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int BUDGET = (227 * 1024) / K::MINB - 2048;
  static constexpr int FIT = BUDGET / (STAGE + 16);
  static constexpr int STAGES = FIT < K::MAXSTAGES ? FIT : K::MAXSTAGES;
  static constexpr int BYTES = 1024 + STAGES * STAGE + 2 * STAGES * 8 + 64;
  static constexpr unsigned TX = (unsigned)(A_BYTES + B_BYTES);
  static_assert(K::BK == 16, "TMA variant assumes 128-byte A rows");   // K tails: TMA zero fill
  static_assert(A_BYTES % 1024 == 0 && (!BKC || B_BYTES % 1024 == 0), "swizzled stages must stay 1024-byte aligned");
  static_assert(STAGES >= 3, "pipeline too shallow");
};

// MULTI: C's M / N index maps through several label groups (dot_decode, e.g. the implicit operand's
// W(p,q,r,s) = X(p,r,L) X(q,s,L): rows (p,r), columns (q,s)); else one stride per side.
template <class K, bool BKC, bool MULTI>
__global__ void __launch_bounds__(K::NTHREADS, K::MINB)
    tt_contract_tma_kernel(const ContractParams p, const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmB) {
  using SM = TmaSmem<K, BKC>;
  constexpr int STAGES = SM::STAGES;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023)) & 1023);   // stays in the shared window (LDS, not generic LD)
  unsigned char* sA = base;                                   // STAGES * A_BYTES
  unsigned char* sB = base + STAGES * SM::A_BYTES;            // STAGES * B_BYTES
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * SM::B_BYTES);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);             // the producer thread's arrive.expect_tx
      mbar_init(&empty[s], K::NMMA);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= K::NMMA) {
    if (warp != K::NMMA || lane != 0) return;
    // ------------------------------------------------------------- TMA producer (one thread)
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    int st = 0;
    unsigned phase = 1;
    for (int64_t wi = blockIdx.x; wi < p.nwork; wi += gridDim.x) {
      const WorkItem w = p.work[wi];
      const CGroupDesc* g = p.groups + w.group;
      const int m0 = g->m_begin + w.mt * K::BM, n0 = g->n_begin + w.nt * K::BN;
      for (int t = g->task_begin; t < g->task_end; ++t) {
        const TaskDesc* td = p.tasks + t;
        const int Kt = td->K;
        // A: [rows][K] view (k tail: out-of-bounds zero fill); B: [rows][K] view ([N][K] blocks) or the
        // [blocks][K][N] view ([K][N] blocks: rows past the block's K are out of bounds, zero fill)
        const int arow = (int)(td->a_off / Kt) + m0;
        const int bsel = BKC ? (int)(td->b_off / Kt) + n0 : (int)(td->b_off / ((int64_t)Kt * p.tma_n));
        for (int k0 = 0; k0 < Kt; k0 += K::BK) {
          mbar_wait_sleep(&empty[st], phase);
          mbar_expect_tx(&full[st], SM::TX);
          tma_load_2d(sA + st * SM::A_BYTES, &tmA, k0, arow, &full[st]);
          if (BKC) tma_load_2d(sB + st * SM::B_BYTES, &tmB, k0, bsel, &full[st]);
          else tma_load_3d(sB + st * SM::B_BYTES, &tmB, n0, k0, bsel, &full[st]);
          if (++st == STAGES) { st = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // --------------------------------------------------------------- MMA warps
  const int wm = warp / K::WN, wn = warp % K::WN;
  const int q = lane & 3, r8 = lane >> 2, pr = perm8(r8);
  const double alpha_ = p.alpha, beta_ = p.beta;
  int st = 0;
  unsigned phase = 0;
  for (int64_t wi = blockIdx.x; wi < p.nwork; wi += gridDim.x) {
    const WorkItem w = p.work[wi];
    const CGroupDesc* g = p.groups + w.group;
    const int m0 = g->m_begin + w.mt * K::BM, n0 = g->n_begin + w.nt * K::BN;
    const int nst = g->nstages;
    double acc[K::MT][K::NT][2];
#pragma unroll
    for (int i = 0; i < K::MT; ++i)
#pragma unroll
      for (int j = 0; j < K::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int s = 0; s < nst; ++s) {
      mbar_wait(&full[st], phase);
      const unsigned char* a = sA + st * SM::A_BYTES;
      const unsigned char* bs = sB + st * SM::B_BYTES;
      const double* b = reinterpret_cast<const double*>(bs);
#pragma unroll
      for (int o = 0; o < K::BK / 8; ++o) {
        double af[K::MT][2], bf[K::NT][2];
#pragma unroll
        for (int i = 0; i < K::MT; ++i) {
          const int m = wm * K::WTM + i * 8 + pr;
          const double2 v =
              *reinterpret_cast<const double2*>(a + m * 128 + ((((4 * o + q) ^ (m & 7))) << 4));
          af[i][0] = v.x;
          af[i][1] = v.y;
        }
#pragma unroll
        for (int j = 0; j < K::NT; ++j) {
          if (BKC) {   // swizzled [n][16 k] rows, fragment columns permuted like A's rows
            const int n = wn * K::WTN + j * 8 + pr;
            const double2 v =
                *reinterpret_cast<const double2*>(bs + n * 128 + ((((4 * o + q) ^ (n & 7))) << 4));
            bf[j][0] = v.x;
            bf[j][1] = v.y;
          } else {
            const int n = wn * K::WTN + j * 8 + r8;
            bf[j][0] = b[(8 * o + 2 * q) * SM::B_LD + n];
            bf[j][1] = b[(8 * o + 2 * q + 1) * SM::B_LD + n];
          }
        }
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int i = 0; i < K::MT; ++i)
#pragma unroll
            for (int j = 0; j < K::NT; ++j) dmma884(acc[i][j], af[i][t], bf[j][t]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == STAGES) { st = 0; phase ^= 1; }
    }
    // epilogue: C row m, column n through one stride per side, or through the label groups (MULTI)
    const bool part = g->flags & kGroupPartial;
    double* Cb = (part ? p.P : p.C) + g->c_off;
    const double alpha = part ? 1.0 : alpha_, beta = part ? 0.0 : beta_;
    const int M = g->M, N = g->N;
    const int32_t cms = g->cm_str[0], cns = g->cn_str[0];
    int32_t mext[kMaxGroup], next[kMaxGroup], cmv[kMaxGroup], cnv[kMaxGroup];
    if (MULTI) {
#pragma unroll
      for (int i = 0; i < kMaxGroup; ++i) {
        mext[i] = g->mext[i];
        next[i] = g->next[i];
        cmv[i] = g->cm_str[i];
        cnv[i] = g->cn_str[i];
      }
    }
#pragma unroll
    for (int i = 0; i < K::MT; ++i) {
      const int m = m0 + wm * K::WTM + i * 8 + pr;
      if (m >= M) continue;
      const int64_t om = MULTI ? (int64_t)dot_decode(m, p.nM, mext, cmv) : (int64_t)m * cms;
#pragma unroll
      for (int j = 0; j < K::NT; ++j) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int n = n0 + wn * K::WTN + j * 8 + (BKC ? perm8(2 * q + r) : 2 * q + r);
          if (n >= N) continue;
          double* c = Cb + om + (MULTI ? (int64_t)dot_decode(n, p.nN, next, cnv) : (int64_t)n * cns);
          const double v = __dmul_rn(alpha, acc[i][j][r]);
          *c = (beta == 0.0) ? v : __fma_rn(beta, *c, v);
        }
      }
    }
  }
}

template <class K, bool BKC, bool MULTI>
static cudaError_t setup_tma_one() {
  return cudaFuncSetAttribute(tt_contract_tma_kernel<K, BKC, MULTI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              TmaSmem<K, BKC>::BYTES);
}
template <class K>
static cudaError_t setup_tma() {
  cudaError_t e;
  if ((e = setup_tma_one<K, false, false>()) != cudaSuccess) return e;
  if ((e = setup_tma_one<K, false, true>()) != cudaSuccess) return e;
  if ((e = setup_tma_one<K, true, false>()) != cudaSuccess) return e;
  return setup_tma_one<K, true, true>();
}
template <class K, bool BKC, bool MULTI>
static cudaError_t launch_tma_one(const ContractParams& p, const CUtensorMap& a, const CUtensorMap& b, int64_t nwork,
                                  cudaStream_t s) {
  const int64_t slots = (int64_t)p.sm_count * K::MINB;
  const unsigned grid = (unsigned)((p.persistent && nwork > slots) ? slots : nwork);
  ContractParams q = p;
  q.nwork = nwork;
  tt_contract_tma_kernel<K, BKC, MULTI><<<grid, K::NTHREADS, TmaSmem<K, BKC>::BYTES, s>>>(q, a, b);
  return cudaGetLastError();
}
// mode bit 0: B is [N][K] (k contiguous); bit 1: multi-group C epilogue
template <class K>
static cudaError_t launch_tma(int mode, const ContractParams& p, const CUtensorMap& a, const CUtensorMap& b,
                              int64_t nwork, cudaStream_t s) {
  switch (mode & 3) {
    case 0: return launch_tma_one<K, false, false>(p, a, b, nwork, s);
    case 1: return launch_tma_one<K, true, false>(p, a, b, nwork, s);
    case 2: return launch_tma_one<K, false, true>(p, a, b, nwork, s);
    default: return launch_tma_one<K, true, true>(p, a, b, nwork, s);
  }
}

template <class K, bool AKC, bool BNC, bool AV, bool BV>
static cudaError_t setup_one() {
  return cudaFuncSetAttribute(tt_contract_ws_kernel<K, AKC, BNC, AV, BV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              Smem<K, AKC, BNC>::BYTES);
}
template <class K, bool AKC, bool BNC>
static cudaError_t setup_orient() {
  cudaError_t e;
  if ((e = setup_one<K, AKC, BNC, true, true>()) != cudaSuccess) return e;
  if ((e = setup_one<K, AKC, BNC, true, false>()) != cudaSuccess) return e;
  if ((e = setup_one<K, AKC, BNC, false, true>()) != cudaSuccess) return e;
  return setup_one<K, AKC, BNC, false, false>();
}
template <class K>
static cudaError_t setup_cfg() {
  cudaError_t e;
  if ((e = setup_orient<K, true, true>()) != cudaSuccess) return e;
  if ((e = setup_orient<K, true, false>()) != cudaSuccess) return e;
  if ((e = setup_orient<K, false, true>()) != cudaSuccess) return e;
  return setup_orient<K, false, false>();
}

template <class K, bool AKC, bool BNC, bool AV, bool BV>
static cudaError_t launch_one(const ContractParams& p, int64_t nwork, cudaStream_t s) {
  // persistent grid: at most the resident CTAs (SM count x CTAs per SM)
  const int64_t slots = (int64_t)p.sm_count * K::MINB;
  const unsigned grid = (unsigned)((p.persistent && nwork > slots) ? slots : nwork);
  ContractParams q = p;
  q.nwork = nwork;
  tt_contract_ws_kernel<K, AKC, BNC, AV, BV><<<grid, K::NTHREADS, Smem<K, AKC, BNC>::BYTES, s>>>(q);
  return cudaGetLastError();
}
template <class K, bool AKC, bool BNC>
static cudaError_t launch_orient(bool av, bool bv, const ContractParams& p, int64_t nwork, cudaStream_t s) {
  if (av && bv) return launch_one<K, AKC, BNC, true, true>(p, nwork, s);
  if (av) return launch_one<K, AKC, BNC, true, false>(p, nwork, s);
  if (bv) return launch_one<K, AKC, BNC, false, true>(p, nwork, s);
  return launch_one<K, AKC, BNC, false, false>(p, nwork, s);
}
template <class K>
static cudaError_t launch_cfg(bool akc, bool bnc, bool av, bool bv, const ContractParams& p, int64_t nwork,
                              cudaStream_t s) {
  if (akc && bnc) return launch_orient<K, true, true>(av, bv, p, nwork, s);
  if (akc) return launch_orient<K, true, false>(av, bv, p, nwork, s);
  if (bnc) return launch_orient<K, false, true>(av, bv, p, nwork, s);
  return launch_orient<K, false, false>(av, bv, p, nwork, s);
}
template <class K>
static VariantInfo info_cfg(const char* name) {
  // shared memory: worst case over orientations
  int smem = Smem<K, true, false>::BYTES;
  if (Smem<K, true, true>::BYTES > smem) smem = Smem<K, true, true>::BYTES;
  if (Smem<K, false, true>::BYTES > smem) smem = Smem<K, false, true>::BYTES;
  if (Smem<K, false, false>::BYTES > smem) smem = Smem<K, false, false>::BYTES;
  return {K::BM, K::BN, K::BK, K::NTHREADS, smem, K::MINB, name};
}

// One translation unit per tile configuration (parallel compilation):
#define TT_WS_DEFINE(NAME, CFG, LABEL)                                                              \
  namespace tt {                                                                                   \
  VariantInfo ws_info_##NAME() { return ws::info_cfg<CFG>(LABEL); }                                \
  cudaError_t ws_setup_##NAME() {                                                                 \
    cudaError_t e = ws::setup_cfg<CFG>();                                                          \
    return e != cudaSuccess ? e : ws::setup_tma<CFG>();                                            \
  }                                                                                                \
  cudaError_t ws_launch_tma_##NAME(int mode, const ContractParams& p, const CUtensorMap& a,       \
                                   const CUtensorMap& b, int64_t nwork, cudaStream_t s) {          \
    return ws::launch_tma<CFG>(mode, p, a, b, nwork, s);                                           \
  }                                                                                                \
  cudaError_t ws_launch_##NAME(bool akc, bool bnc, bool av, bool bv, const ContractParams& p,      \
                               int64_t nwork, cudaStream_t s) {                                    \
    return ws::launch_cfg<CFG>(akc, bnc, av, bv, p, nwork, s);                                     \
  }                                                                                                \
  }

}  // namespace ws

}  // namespace tt
