// tt_triples.cu -- sm_100a kernels of the perturbative-triples path (PAPER Eqs. cc14,
// tensort, abt, tensort2, P343-413).
//
// retile_kernel: copies of the inputs in dense, permuted layouts (global index -> source block).
//
// triples_fused_kernel: one CTA per (occupied triple i<j<k, virtual box triple) unit.  The 18 terms of
// Eq. tensort regroup exactly into three GEMMs over the same box (reading R27 for the sixth sign):
//     W(a,b,c) = G(a; b,c) - G(b; a,c) + G(c; a,b)
//     G(r; p,q) = sum_s sigma_s sum_m v^{x_s y_s}_{m r} t^{m z_s}_{p q}      (terms 1,4,7 / 2,5,8 / 3,6,9)
//               - sum_s sigma_s sum_e t^{y_s z_s}_{e r} v^{e x_s}_{p q}       (terms 12,15,18 / 11,14,17 / 10,13,16)
// with (x,y,z,sigma) = (i,j,k,+), (i,k,j,-), (j,k,i,+) for the m sums and (x; y,z) = (i; j,k), (j; i,k),
// (k; i,j) with signs (-,+,-) for the e sums.  Each G is a DMMA GEMM (rows r in the box, columns the
// (p,q) box pairs, K = 3 n_o + 3 n_v) staged by cp.async; its accumulators are folded into a 16^3 cube in
// shared memory, and the energy of Eq. cc14, (W + V1) W / D over a<b<c (V1 = Eq. tensort2), is reduced
// in the same CTA.  W never reaches HBM.
#include <cuda.h>

#include <algorithm>

#include "tt_launch.h"

namespace tt {

namespace {

__device__ __forceinline__ void cpa16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 16 : 0;   // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

constexpr int BX = kTripBox;        // box edge
constexpr int KC = 8;               // k rows per stage
constexpr int NS = 4;               // stages
constexpr int PS = BX + 4;          // P row stride (doubles): = 4 mod 16 -> conflict-free A fragments
constexpr int QS = BX * BX + 4;     // Q row stride: = 4 mod 16 -> conflict-free B fragments
constexpr int THREADS = 256;
constexpr int NWARP = THREADS / 32;
constexpr int CW = BX * BX / NWARP;            // GEMM columns per warp
constexpr int NFR = CW / 8;                    // 8-wide column fragments per warp
constexpr int NQ = KC * 128 / THREADS;         // Q rows copied per thread per stage
constexpr int QR = THREADS / 128;              // row step between them

// W cube (a, b, c) in shared memory with the innermost index XOR-swizzled by f(a) ^ f(b): the fold of each
// GEMM (lanes spread over {row} x {even or odd columns}) and the energy loop are then bank-conflict free
__device__ __forceinline__ int swz(int x) { return (x & 1) | ((x & 2) << 2) | (x & 4); }
__device__ __forceinline__ int cidx(int a, int b, int c) { return (a * BX + b) * BX + (c ^ swz(a) ^ swz(b)); }

}  // namespace

// dst block element e -> global coordinates (dst dim order) -> the src block (another tiling and order)
__global__ void retile_kernel(const RetileParams p) {
  const Segment sg = p.segs[blockIdx.x];
  const RetileBlk b = p.blks[sg.desc];
  double* dst = p.dst + b.dst_off;
  for (int64_t e = sg.e0 + threadIdx.x; e < sg.e1; e += blockDim.x) {
    int64_t r = e;
    int32_t g[TT_MAX_ORDER];
    for (int q = p.order - 1; q >= 0; --q) {
      const int64_t x = b.ext[q];
      g[q] = b.org[q] + (int32_t)(r % x);
      r /= x;
    }
    int64_t bid = 0, el = 0;
    for (int q = 0; q < p.order; ++q) {
      const int32_t gq = g[p.sdim[q]];
      const int32_t t = p.g2t[q][gq];
      const int64_t o0 = p.toff[q][t];
      bid = bid * p.sgrid[q] + t;
      el = el * (p.toff[q][t + 1] - o0) + (gq - o0);
    }
    const int64_t so = p.sblk_off[bid];
    dst[e] = so >= 0 ? p.src[so + el] : 0.0;
  }
}

// dense copies (rt) -> blocked, pre-swizzled copies of the default kernel (see TriplesParams)
__device__ __forceinline__ int32_t unpad_row(int32_t kq, int32_t half, int32_t k2, int32_t n) {
  // padded row -> summed index, -1 for a padding row
  const int32_t k = kq < k2 ? kq : half + (kq - k2);
  return (kq < k2 ? k < half : k < n) ? k : -1;
}

__global__ void blockify_kernel(int mode, const TriplesParams p, double* __restrict__ dst, int64_t n) {
  const int32_t nO = p.nO, nV = p.nV, nb = p.nb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (mode <= 1) {   // [o][bp][bq][k'/8][p][k'%8][q]
      const int32_t kp = mode == 0 ? p.kpo : p.kpv;
      int64_t r = e;
      const int qs = (int)(r % BX); r /= BX;
      const int k8 = (int)(r % KC); r /= KC;
      const int pl = (int)(r % BX); r /= BX;
      const int32_t kst = (int32_t)(r % (kp / KC)); r /= kp / KC;
      const int32_t bq = (int32_t)(r % nb); r /= nb;
      const int32_t bp = (int32_t)(r % nb); r /= nb;
      const int32_t o = (int32_t)r;
      const int32_t kq = kst * KC + k8;
      const int32_t k = mode == 0 ? unpad_row(kq, p.o_half, p.ko2, nO) : unpad_row(kq, p.v_half, p.kv2, nV);
      const int ql = qs ^ ((kq & 3) << 2);   // stored at column q ^ 4(k' mod 4)
      const int32_t pv = p.box_lo[bp] + pl, qv = p.box_lo[bq] + ql;
      if (pl < p.box_ext[bp] && ql < p.box_ext[bq] && k >= 0)
        v = mode == 0 ? p.T2[(((int64_t)k * nO + o) * nV + pv) * nV + qv]      // T2[m][z][p][q]
                      : p.VV[(((int64_t)k * nO + o) * nV + pv) * nV + qv];     // VV[e][x][p][q]
    } else {           // [o1][o2][br][k'][16]
      const int32_t kp = mode == 2 ? p.kpo : p.kpv;
      int64_t r = e;
      const int rs = (int)(r % BX); r /= BX;
      const int32_t kq = (int32_t)(r % kp); r /= kp;
      const int32_t br = (int32_t)(r % nb); r /= nb;
      const int32_t o2 = (int32_t)(r % nO); r /= nO;
      const int32_t o1 = (int32_t)r;
      const int32_t k = mode == 2 ? unpad_row(kq, p.o_half, p.ko2, nO) : unpad_row(kq, p.v_half, p.kv2, nV);
      const int rl = rs ^ ((kq & 3) << 2);
      const int32_t rv = p.box_lo[br] + rl;
      if (rl < p.box_ext[br] && k >= 0)
        v = mode == 2 ? p.VO[(((int64_t)o1 * nO + o2) * nO + k) * nV + rv]     // VO[x][y][m][r]
                      : p.T2[(((int64_t)o1 * nO + o2) * nV + k) * nV + rv];    // T2[y][z][e][r]
    }
    dst[e] = v;
  }
}

cudaError_t launch_blockify(int mode, const TriplesParams& p, double* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 64);
  blockify_kernel<<<(unsigned)blocks, 256, 0, s>>>(mode, p, dst, n);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(THREADS, 2) triples_fused_kernel(const TriplesParams p) {
  extern __shared__ __align__(16) double sm[];
  double* Ps = sm;                              // [NS][KC][PS]
  double* Qs = Ps + NS * KC * PS;               // [NS][KC][QS]
  double* cube = Qs + NS * KC * QS;             // [BX][BX][BX]  (a, b, c)
  double* red = cube + BX * BX * BX;            // [THREADS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t u = p.unit0 + blockIdx.x;
  const int2 un = p.units[u];
  const int4 bx = p.box3[un.x];
  const int4 tr = p.trip[un.y];
  const int32_t nO = p.nO, nV = p.nV;
  const int32_t lo[3] = {p.box_lo[bx.x], p.box_lo[bx.y], p.box_lo[bx.z]};
  const int32_t ex[3] = {p.box_ext[bx.x], p.box_ext[bx.y], p.box_ext[bx.z]};
  const int32_t I = tr.x, J = tr.y, K = tr.z;
  const int32_t kA = 3 * nO, kT = 3 * nO + 3 * nV;
  const int32_t nst = (kT + KC - 1) / KC;       // stages per GEMM
  const int32_t total = 3 * nst;
  const int64_t sQ = (int64_t)nO * nV * nV;     // Q row step per k inside a segment (both parts)

  // Copy assignment (fixed per thread): Q = KC rows x BX p x BX/2 pairs = NQ copies per thread (rows
  // qrow + QR n), P = KC rows x BX/2 pairs for threads < 64.  Each copied k row keeps a cursor
  // (pointer, step per k, end of its segment); the division-based address math runs only when a row
  // crosses a segment (or GEMM) boundary.
  const int qp = (tid & 127) >> 3, qq = 2 * (tid & 7), qrow = tid >> 7;   // a warp fills 512 contiguous bytes
  static_assert(THREADS % 128 == 0 && KC * (BX / 2) <= THREADS, "copy mapping");
  const int prow = tid >> 3, pr2 = 2 * (tid & 7);
  const bool has_p = tid < KC * (BX / 2);
  // per GEMM box roles: g = 0 -> (a; b,c), 1 -> (b; a,c), 2 -> (c; a,b)
  int32_t lr = 0, lp = 0, lq = 0;
  bool okr = false, okpq = false;
  auto set_gemm = [&](int g) {
    const int32_t lo_r = g == 0 ? lo[0] : (g == 1 ? lo[1] : lo[2]);
    const int32_t ex_r = g == 0 ? ex[0] : (g == 1 ? ex[1] : ex[2]);
    const int32_t lo_p = g == 0 ? lo[1] : lo[0], ex_p = g == 0 ? ex[1] : ex[0];
    const int32_t lo_q = g == 2 ? lo[1] : lo[2], ex_q = g == 2 ? ex[1] : ex[2];
    lr = lo_r + pr2;
    lp = lo_p + qp;
    lq = lo_q + qq;
    okr = pr2 < ex_r;
    okpq = qp < ex_p && qq < ex_q;
  };
  // source of P row kap (this thread's pair pr2) and its step / segment end
  auto p_src = [&](int32_t kap, const double*& ptr, int64_t& step, int32_t& end) {
    if (kap < kA) {
      const int s = kap / nO, m = kap - s * nO;
      const int32_t x = (s == 2) ? J : I, y = (s == 0) ? J : K;
      ptr = p.VO + (((int64_t)x * nO + y) * nO + m) * nV + lr;
      step = nV;
      end = (s + 1) * nO;
    } else if (kap < kT) {
      const int32_t kb = kap - kA;
      const int s = kb / nV, e = kb - s * nV;
      const int32_t y = (s == 0) ? J : I, z = (s == 2) ? J : K;
      ptr = p.T2 + (((int64_t)y * nO + z) * nV + e) * nV + lr;
      step = nV;
      end = kA + (s + 1) * nV;
    } else {
      ptr = nullptr;
      step = 0;
      end = 0x7fffffff;
    }
  };
  auto q_src = [&](int32_t kap, const double*& ptr, int32_t& end) {
    if (kap < kA) {
      const int s = kap / nO, m = kap - s * nO;
      const int32_t z = (s == 0) ? K : (s == 1 ? J : I);
      ptr = p.T2 + (((int64_t)m * nO + z) * nV + lp) * nV + lq;
      end = (s + 1) * nO;
    } else if (kap < kT) {
      const int32_t kb = kap - kA;
      const int s = kb / nV, e = kb - s * nV;
      const int32_t x = (s == 0) ? I : (s == 1 ? J : K);
      ptr = p.VV + (((int64_t)e * nO + x) * nV + lp) * nV + lq;
      end = kA + (s + 1) * nV;
    } else {
      ptr = nullptr;
      end = 0x7fffffff;
    }
  };
  const double* pptr = nullptr;
  int64_t pstep = 0;
  int32_t pend = 0, pkap = 0;
  const double* qptr[NQ];
  int32_t qend[NQ], qkap[NQ];

  // issue the copies of the next stage (stages are issued in order; counters instead of divisions)
  int ig = 0, ik0 = 0, islot = 0;
  auto issue = [&]() {
    const int g = ig;
    const int32_t k0 = ik0;
    double* P = Ps + islot * KC * PS;
    double* Q = Qs + islot * KC * QS;
    if (k0 == 0) {   // new GEMM: roles and cursors from scratch
      set_gemm(g);
      pkap = prow;
      p_src(pkap, pptr, pstep, pend);
#pragma unroll
      for (int n = 0; n < NQ; ++n) {
        qkap[n] = qrow + QR * n;
        q_src(qkap[n], qptr[n], qend[n]);
      }
    } else {
      pkap += KC;
      if (pkap >= pend) p_src(pkap, pptr, pstep, pend);
      else pptr += KC * pstep;
#pragma unroll
      for (int n = 0; n < NQ; ++n) {
        qkap[n] += KC;
        if (qkap[n] >= qend[n]) q_src(qkap[n], qptr[n], qend[n]);
        else qptr[n] += KC * sQ;
      }
    }
    if (has_p) {
      const bool ok = okr && pptr != nullptr;
      cpa16(P + prow * PS + pr2, ok ? (const void*)pptr : (const void*)p.VO, ok);
    }
#pragma unroll
    for (int n = 0; n < NQ; ++n) {
      const bool ok = okpq && qptr[n] != nullptr;
      cpa16(Q + (qrow + QR * n) * QS + qp * BX + qq, ok ? (const void*)qptr[n] : (const void*)p.T2, ok);
    }
    islot = (islot + 1 == NS) ? 0 : islot + 1;
    ik0 += KC;
    if (ik0 >= nst * KC) { ik0 = 0; ++ig; }
  };

  double acc[2][NFR][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int f = 0; f < NFR; ++f) acc[a][f][0] = acc[a][f][1] = 0.0;

#pragma unroll 1
  for (int t = 0; t < NS - 1; ++t) {
    if (t < total) issue();
    cpa_commit();
  }
  int g = 0, k0 = 0, slot = 0;
#pragma unroll 1
  for (int t = 0; t < total; ++t) {
    cpa_wait<NS - 2>();
    __syncthreads();
    if (t + NS - 1 < total) issue();
    cpa_commit();
    const double* P = Ps + slot * KC * PS;
    const double* Q = Qs + slot * KC * QS;
    slot = (slot + 1 == NS) ? 0 : slot + 1;
#pragma unroll
    for (int kk = 0; kk < KC / 4; ++kk) {
      const int kl = kk * 4 + (lane & 3);
      const int32_t kap = k0 + kl;
      // sign of this k row: m sums (+,-,+), e sums (-,+,-)
      bool neg;
      if (kap < kA) neg = (kap >= nO && kap < 2 * nO);
      else neg = !(kap - kA >= nV && kap - kA < 2 * nV);
      const long long sg = neg ? (long long)0x8000000000000000ull : 0ll;   // sign bit flip (integer pipe)
      const double a0 = __longlong_as_double(__double_as_longlong(P[kl * PS + (lane >> 2)]) ^ sg);
      const double a1 = __longlong_as_double(__double_as_longlong(P[kl * PS + 8 + (lane >> 2)]) ^ sg);
#pragma unroll
      for (int f = 0; f < NFR; ++f) {
        const double b = Q[kl * QS + warp * CW + f * 8 + (lane >> 2)];
        dmma(acc[0][f], a0, b);
        dmma(acc[1][f], a1, b);
      }
    }
    k0 += KC;
    if (k0 >= nst * KC) {                    // GEMM g done: fold into the cube
      __syncthreads();
#pragma unroll
      for (int rf = 0; rf < 2; ++rf)
#pragma unroll
        for (int f = 0; f < NFR; ++f)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = rf * 8 + (lane >> 2);
            const int col = warp * CW + f * 8 + 2 * (lane & 3) + h;
            const int pp = col / BX, q = col % BX;
            const double v = acc[rf][f][h];
            if (g == 0) cube[cidx(row, pp, q)] = v;
            else if (g == 1) cube[cidx(pp, row, q)] -= v;
            else cube[cidx(pp, q, row)] += v;
            acc[rf][f][h] = 0.0;
          }
      k0 = 0;
      ++g;
    }
  }
  cpa_wait<0>();
  __syncthreads();
  // Eq. cc14 over the cube: (W + V1) W / D for a<b<c (i<j<k by construction)
  double s = 0.0;
  const double dijk = p.eps_o[I] + p.eps_o[J] + p.eps_o[K];
  for (int idx = tid; idx < BX * BX * BX; idx += THREADS) {
    const int la = idx / (BX * BX), lb = (idx / BX) % BX, lc = idx % BX;
    if (la >= ex[0] || lb >= ex[1] || lc >= ex[2]) continue;
    const int32_t a = lo[0] + la, b = lo[1] + lb, c = lo[2] + lc;
    if (!(a < b && b < c)) continue;
    const double W = cube[cidx(la, lb, lc)];
    // V1 (Eq. tensort2): pairs (x,y;z) = (i,j;k)+, (i,k;j)-, (j,k;i)+  x  (p,q;r) = (a,b;c)+, (a,c;b)-, (b,c;a)+
    double v1 = 0.0;
    const int32_t ox[3] = {I, I, J}, oy[3] = {J, K, K}, oz[3] = {K, J, I};
    const int32_t vp[3] = {a, a, b}, vq[3] = {b, c, c}, vr[3] = {c, b, a};
#pragma unroll
    for (int pr = 0; pr < 3; ++pr) {
      double inner = 0.0;
#pragma unroll
      for (int pq = 0; pq < 3; ++pq) {
        const double term = p.VD[(((int64_t)ox[pr] * nO + oy[pr]) * nV + vp[pq]) * nV + vq[pq]] *
                            p.T1[(int64_t)vr[pq] * nO + oz[pr]];
        inner = (pq == 1) ? inner - term : inner + term;
      }
      v1 = (pr == 1) ? v1 - inner : v1 + inner;
    }
    const double D = dijk - p.eps_v[a] - p.eps_v[b] - p.eps_v[c];
    s += (W + v1) * W / D;
  }
  red[tid] = s;
  __syncthreads();
  for (int o = THREADS / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (tid == 0) p.partials[u] = red[0];
}

// -------------------------------------------------------------------------------------------------
// TMA variant: one thread issues, per stage, two 4-D cp.async.bulk.tensor boxes (P: 20 r x 8 k; Q:
// 18 q x 18 p x 8 k) that complete on the stage's mbarrier.  The boxes are 2 wider than the data so
// that the shared-memory row strides (20 and 18 x 18 = 324 doubles, both = 4 mod 16) keep the DMMA
// fragment loads conflict-free; their extra columns and the tail boxes' columns beyond the box extents
// are computed and never read back; k rows beyond a segment (m >= n_o, e >= n_v) are TMA zero fill, so
// every stage lies inside one segment (uniform sign) and no per-thread address arithmetic remains.
namespace {
constexpr int TPW = BX + 4;                 // P box width (r)
constexpr int TQW = BX + 2;                 // Q box width (q) and height (p)
constexpr int TQS = TQW * TQW;              // Q k-row stride (324 = 4 mod 16)
constexpr int TNS = 3;                      // stages
constexpr int TP_BYTES = KC * TPW * 8;      // 1280
constexpr int TQ_BYTES = KC * TQS * 8;      // 20736
constexpr int TSTAGE = TP_BYTES + TQ_BYTES;

// default kernel: 1-D bulk copies of the blocked copies, Q (8 x 16 x 16) then P (8 x 16) per stage
constexpr int BQ_BYTES = KC * BX * BX * 8;   // 16384
constexpr int BP_BYTES = KC * BX * 8;        // 1024
constexpr int BSTAGE = BQ_BYTES + BP_BYTES;
constexpr int BNS = 4;                       // stages

__device__ __forceinline__ void tbar_init(uint64_t* bar, unsigned count) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s), "r"(count));
}
__device__ __forceinline__ void tbar_expect(uint64_t* bar, unsigned bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tbar_wait(uint64_t* bar, unsigned parity) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n"
      "TWAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TWAIT_%=;\n}\n" ::"r"(s),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(d), "l"(gmem), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void tma4(void* smem, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
      ::"r"(d), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b)
      : "memory");
}
}  // namespace

// One more warp than the compute warps: warp 8 is the TMA producer (lane 0 issues the boxes of every
// stage into a TNS-slot ring; per-slot "full" barriers complete on the transaction bytes, per-slot
// "empty" barriers collect one arrival per compute warp), so no CTA-wide barrier sits in the k loop.
constexpr int TTHREADS = THREADS + 32;

// Whether the 8x8 output fragment (rows r0..r0+7 of the GEMM's row box, column pair (p, q0..q0+7)) of GEMM
// g holds an element with a < b < c inside the boxes' extents (roles: g = 0 (a; b,c), 1 (b; a,c),
// 2 (c; a,b)).  Greedy: the smallest a, then the smallest b > a, then the smallest c > b.
__device__ __forceinline__ bool frag_needed(int g, int r0, int pp, int q0, const int32_t* lo, const int32_t* ex) {
  // interval of virtual index d (0 = a, 1 = b, 2 = c): the row role (r0..r0+7) is d == g, the column-pair
  // role (pp) is b for g = 0 and a otherwise, the inner column role (q0..q0+7) the remaining index;
  // written without local arrays (no stack traffic)
  auto iv = [&](int d, int& gl, int& gh) {
    int s, e;
    if (d == g) { s = r0; e = r0 + 8; }
    else if (d == (g == 0 ? 1 : 0)) { s = pp; e = pp + 1; }
    else { s = q0; e = q0 + 8; }
    const int h = e < ex[d] ? e : ex[d];
    gl = lo[d] + s;
    gh = lo[d] + h - 1;
    return s < h;
  };
  int l0, h0, l1, h1, l2, h2;
  if (!iv(0, l0, h0) || !iv(1, l1, h1) || !iv(2, l2, h2)) return false;
  const int b = (l0 + 1 > l1) ? l0 + 1 : l1;   // smallest a, then the smallest b > a, c > b
  if (b > h1) return false;
  const int c = (b + 1 > l2) ? b + 1 : l2;
  return c <= h2;
}

__device__ __forceinline__ void tbar_arrive(uint64_t* bar) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(s) : "memory");
}
__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(THREADS) : "memory"); }

// One segment of a GEMM in the default kernel: n stages of 8 k rows.  The warp's column slots are NB
// fragments needing both row halves, then N0 needing the first, then N1 needing the second (all
// compile-time), so fewer needed fragments issue fewer DMMAs instead of predicated-off ones.
template <int NB, int N0, int N1>
__device__ __forceinline__ void seg_mma(double (&acc)[2][NFR][2], int n, int& slot, unsigned& phase,
                                        unsigned char* base, uint64_t* full, uint64_t* empty,
                                        const int (&qa)[NFR], int sw, long long sgm, int lane) {
  constexpr int NS = NB + N0 + N1;
#pragma unroll 1
  for (int jj = 0; jj < n; ++jj) {
    tbar_wait(&full[slot], phase);
    if (NS > 0) {
      const double* Q = reinterpret_cast<const double*>(base + slot * BSTAGE);
      const double* P = reinterpret_cast<const double*>(base + slot * BSTAGE + BQ_BYTES);
#pragma unroll
      for (int kk = 0; kk < KC / 4; ++kk) {
        const int kl = kk * 4 + (lane & 3);
        const double a0 = NB + N0 == 0 ? 0.0
            : __longlong_as_double(__double_as_longlong(P[kl * BX + ((lane >> 2) ^ sw)]) ^ sgm);
        const double a1 = NB + N1 == 0 ? 0.0
            : __longlong_as_double(__double_as_longlong(P[kl * BX + ((8 + (lane >> 2)) ^ sw)]) ^ sgm);
#pragma unroll
        for (int f = 0; f < NS; ++f) {
          const double b = Q[kk * 4 * BX + qa[f]];
          if (f < NB + N0) dmma(acc[0][f], a0, b);
          if (f < NB || f >= NB + N0) dmma(acc[1][f], a1, b);
        }
      }
    }
    __syncwarp();
    if (lane == 0) tbar_arrive(&empty[slot]);
    if (++slot == BNS) { slot = 0; phase ^= 1; }
  }
}

__global__ void __launch_bounds__(TTHREADS, 2)
    triples_fused_tma_kernel(const TriplesParams p) {
  extern __shared__ __align__(128) unsigned char tsm_raw[];
  unsigned char* base = tsm_raw + ((128 - ((unsigned)__cvta_generic_to_shared(tsm_raw) & 127)) & 127);   // stays in the shared window (LDS, not generic LD)
  double* cube = reinterpret_cast<double*>(base + BNS * BSTAGE);   // [BX][BX][BX]
  double* red = cube + BX * BX * BX;                               // [THREADS]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + THREADS);     // [BNS]
  uint64_t* empty = full + BNS;                                    // [BNS]
  int32_t* segb = reinterpret_cast<int32_t*>(empty + BNS);         // [3][6] first summed index
  int32_t* segn = segb + 18;                                       // [3][6] stages
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t u = p.unit0 + blockIdx.x;
  const int2 un = p.units[u];
  const int4 bx = p.box3[un.x];
  const int4 tr = p.trip[un.y];
  const int32_t nO = p.nO, nV = p.nV;
  const int32_t lo[3] = {p.box_lo[bx.x], p.box_lo[bx.y], p.box_lo[bx.z]};
  const int32_t ex[3] = {p.box_ext[bx.x], p.box_ext[bx.y], p.box_ext[bx.z]};
  const int32_t I = tr.x, J = tr.y, K = tr.z;
  if (tid == 0) {
    for (int q = 0; q < BNS; ++q) {
      tbar_init(&full[q], 1);
      tbar_init(&empty[q], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < 18) {
    // summed range of segment sg of GEMM g.  With spin (R6: alpha = first half), the m of v^{xy}_{m r}
    // must have spin s_x + s_y - s_r and the e of v^{e x}_{p q} spin s_p + s_q - s_x (R7 maps); the other
    // half of the sum is identically zero and is skipped.
    const int g = tid / 6, sg = tid % 6;
    const int32_t oh = p.o_half, vh = p.v_half;
    auto so = [&](int32_t x) { return oh ? (x < oh ? 1 : -1) : 0; };
    auto sv = [&](int32_t v) { return vh ? (v < vh ? 1 : -1) : 0; };
    const int32_t sr = sv(g == 0 ? lo[0] : (g == 1 ? lo[1] : lo[2]));
    const int32_t sp = sv(g == 0 ? lo[1] : lo[0]), sq = sv(g == 2 ? lo[1] : lo[2]);
    int32_t b = 0, e = 0;
    if (sg < 3) {
      const int32_t x = (sg == 2) ? J : I, y = (sg == 0) ? J : K;
      const int32_t sm = so(x) + so(y) - sr;
      if (!oh) { b = 0; e = nO; }
      else if (sm == 1) { b = 0; e = oh; }
      else if (sm == -1) { b = oh; e = nO; }
    } else {
      const int32_t x = (sg == 3) ? I : (sg == 4 ? J : K);
      const int32_t se = sp + sq - so(x);
      if (!vh) { b = 0; e = nV; }
      else if (se == 1) { b = 0; e = vh; }
      else if (se == -1) { b = vh; e = nV; }
    }
    segb[tid] = b;
    segn[tid] = (e - b + KC - 1) / KC;
  }
  __syncthreads();

  if (warp == NWARP) {
    // ---------------------------------------------------------------- TMA producer (one thread)
    if (lane != 0) return;
    int slot = 0;
    unsigned phase = 1;   // empty barriers: the first pass over the ring does not wait
    const int32_t nb = p.nb, kpo = p.kpo, kpv = p.kpv;
    for (int g = 0; g < 3; ++g) {
      const int32_t br = g == 0 ? bx.x : (g == 1 ? bx.y : bx.z);   // box ids of the roles (r; p, q)
      const int32_t bp = g == 0 ? bx.y : bx.x;
      const int32_t bq = g == 2 ? bx.y : bx.z;
      for (int sg = 0; sg < 6; ++sg) {
        const int32_t n = segn[g * 6 + sg];
        for (int jj = 0; jj < n; ++jj) {
          // padded first row: segments start at 0 or at the second spin range
          const int32_t k0 = (segb[g * 6 + sg] == 0 ? 0 : (sg < 3 ? p.ko2 : p.kv2)) + jj * KC;
          const unsigned qbytes = (unsigned)p.box_ext[bp] * (KC * BX * 8);   // ext_p rows of p
          tbar_wait(&empty[slot], phase);
          unsigned char* st = base + slot * BSTAGE;
          tbar_expect(&full[slot], qbytes + (unsigned)BP_BYTES);
          const double *qsrc, *psrc;
          if (sg < 3) {
            const int32_t x = (sg == 2) ? J : I, y = (sg == 0) ? J : K, z = (sg == 0) ? K : (sg == 1 ? J : I);
            qsrc = p.QT2 + ((((int64_t)z * nb + bp) * nb + bq) * kpo + k0) * (BX * BX);   // T2[m][z][p][q]
            psrc = p.PVO + ((((int64_t)x * nO + y) * nb + br) * kpo + k0) * BX;          // VO[x][y][m][r]
          } else {
            const int s3 = sg - 3;
            const int32_t x = (s3 == 0) ? I : (s3 == 1 ? J : K), y = (s3 == 0) ? J : I, z = (s3 == 2) ? J : K;
            qsrc = p.QVV + ((((int64_t)x * nb + bp) * nb + bq) * kpv + k0) * (BX * BX);   // VV[e][x][p][q]
            psrc = p.PT2 + ((((int64_t)y * nO + z) * nb + br) * kpv + k0) * BX;          // T2[y][z][e][r]
          }
          bulk_copy(st, qsrc, qbytes, &full[slot]);
          bulk_copy(st + BQ_BYTES, psrc, BP_BYTES, &full[slot]);
          if (++slot == BNS) { slot = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ compute warps (8)
  double acc[2][NFR][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int f = 0; f < NFR; ++f) acc[a][f][0] = acc[a][f][1] = 0.0;
  int slot = 0;
  unsigned phase = 0;
#pragma unroll 1
  for (int g = 0; g < 3; ++g) {
    // the 8-column output fragments that hold a needed W(a,b,c) (a<b<c inside the extents), in three
    // classes -- both row halves, the first only, the second only -- listed in that order and dealt
    // round-robin to the warps: no warp holds more than ceil(n/8) of them, each warp's slots run
    // both -> first -> second, and the slot counts per class (nb_, n0_, n1_) select a compile-time loop
    // (diagonal box triples and narrow tail boxes issue fewer DMMAs, not predicated-off ones)
    uint32_t colp = 0xffffffffu;   // slot f: column fragment (colp >> 8f) & 0xff, 0xff = none
    int nb_ = 0, n0_ = 0, n1_ = 0;
    {
      const int col = lane * 8;                 // lane c tests column fragment c
      const uint32_t m0 = __ballot_sync(0xffffffffu, frag_needed(g, 0, col / BX, col % BX, lo, ex));
      const uint32_t m1 = __ballot_sync(0xffffffffu, frag_needed(g, 8, col / BX, col % BX, lo, ex));
      const uint32_t cb = m0 & m1, c0 = m0 & ~m1, c1 = m1 & ~m0;
      const int kb = __popc(cb), k0 = kb + __popc(c0), kn = k0 + __popc(c1);
#pragma unroll
      for (int f = 0; f < NFR; ++f) {
        const int k = f * NWARP + warp;         // this slot takes the k-th needed fragment
        if (k < kn) {
          const uint32_t c = k < kb ? __fns(cb, 0, k + 1) : (k < k0 ? __fns(c0, 0, k - kb + 1) : __fns(c1, 0, k - k0 + 1));
          colp = (colp & ~(0xffu << (8 * f))) | (c << (8 * f));
          if (k < kb) ++nb_; else if (k < k0) ++n0_; else ++n1_;
        }
      }
    }
#pragma unroll 1
    for (int sg = 0; sg < 6; ++sg) {
      const int32_t n = segn[g * 6 + sg];
      const bool neg = sg < 3 ? sg == 1 : sg != 4;   // m sums (+,-,+), e sums (-,+,-)
      const long long sgm = neg ? (long long)0x8000000000000000ull : 0ll;
      // every stage starts at a padded row = 0 mod 8: the swizzle is (k' mod 4) = the lane's k row
      const int sw = (lane & 3) << 2;                               // columns XOR 4(k' mod 4)
      int qa[NFR];                                                  // Q offsets ([p][k'%8][q]) of this lane
#pragma unroll
      for (int f = 0; f < NFR; ++f) {
        const int col = (int)((colp >> (8 * f)) & 31u) * 8 + (lane >> 2);
        qa[f] = (col / BX) * (KC * BX) + (lane & 3) * BX + ((col % BX) ^ sw);
      }
      switch (nb_ * 25 + n0_ * 5 + n1_) {
#define TT_SEG(B_, F_, S_) \
  case B_ * 25 + F_ * 5 + S_: seg_mma<B_, F_, S_>(acc, n, slot, phase, base, full, empty, qa, sw, sgm, lane); break;
        TT_SEG(0, 0, 1) TT_SEG(0, 0, 2) TT_SEG(0, 0, 3) TT_SEG(0, 0, 4) TT_SEG(0, 1, 0)
        TT_SEG(0, 1, 1) TT_SEG(0, 1, 2) TT_SEG(0, 1, 3) TT_SEG(0, 2, 0) TT_SEG(0, 2, 1)
        TT_SEG(0, 2, 2) TT_SEG(0, 3, 0) TT_SEG(0, 3, 1) TT_SEG(0, 4, 0) TT_SEG(1, 0, 0)
        TT_SEG(1, 0, 1) TT_SEG(1, 0, 2) TT_SEG(1, 0, 3) TT_SEG(1, 1, 0) TT_SEG(1, 1, 1)
        TT_SEG(1, 1, 2) TT_SEG(1, 2, 0) TT_SEG(1, 2, 1) TT_SEG(1, 3, 0) TT_SEG(2, 0, 0)
        TT_SEG(2, 0, 1) TT_SEG(2, 0, 2) TT_SEG(2, 1, 0) TT_SEG(2, 1, 1) TT_SEG(2, 2, 0)
        TT_SEG(3, 0, 0) TT_SEG(3, 0, 1) TT_SEG(3, 1, 0) TT_SEG(4, 0, 0)
#undef TT_SEG
        default: seg_mma<0, 0, 0>(acc, n, slot, phase, base, full, empty, qa, sw, sgm, lane); break;
      }
    }
    // GEMM g done: fold into the cube (each cube entry has one owner thread per GEMM; the barriers
    // order the three folds)
    // (cube entries outside every needed fragment are never written and never read)
#pragma unroll
    for (int f = 0; f < NFR; ++f) {
      if (((colp >> (8 * f)) & 0xffu) == 0xffu) continue;
#pragma unroll
      for (int rf = 0; rf < 2; ++rf)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = rf * 8 + (lane >> 2);
          const int col = (int)((colp >> (8 * f)) & 31u) * 8 + 2 * (lane & 3) + h;
          const int pp = col / BX, q = col % BX;
          const double v = acc[rf][f][h];
          if (g == 0) cube[cidx(row, pp, q)] = v;
          else if (g == 1) cube[cidx(pp, row, q)] -= v;
          else cube[cidx(pp, q, row)] += v;
          acc[rf][f][h] = 0.0;
        }
    }
    compute_sync();
  }
  // Eq. cc14 over the cube.  The V1 inputs of the unit (Eq. tensort2: v^{xy}_{pq} over the 3 occupied
  // pairs x 3 virtual box pairs, t^z_r over the 3 boxes x 3 occupied, eps_v of the boxes) are first
  // staged in the (now free) stage buffers with coalesced loads, so the element loop reads shared
  // memory only.
  constexpr int VDP = BX + 1;                                       // padded tile row
  double* vds = reinterpret_cast<double*>(base);                    // [3 pr][3 pq][BX][VDP]
  double* t1s = vds + 9 * BX * VDP;                                 // [3 box][BX][3 z]
  double* epv = t1s + 3 * BX * 3;                                   // [3 box][BX]
  {
    // selects instead of indexed local arrays (register resident)
    auto box_lo = [&](int i) { return i == 0 ? lo[0] : (i == 1 ? lo[1] : lo[2]); };
    auto box_ex = [&](int i) { return i == 0 ? ex[0] : (i == 1 ? ex[1] : ex[2]); };
    for (int e = tid; e < 9 * BX * BX; e += THREADS) {
      const int t = e / (BX * BX), rr = (e / BX) % BX, cc = e % BX;
      const int pr = t / 3, pq = t % 3;
      const int pbx = pq == 2 ? 1 : 0, qbx = pq == 0 ? 1 : 2;     // (a,b), (a,c), (b,c)
      const int32_t ox = pr == 2 ? J : I, oy = pr == 0 ? J : K;    // (i,j), (i,k), (j,k)
      vds[(t * BX + rr) * VDP + cc] = (rr < box_ex(pbx) && cc < box_ex(qbx))
          ? p.VD[(((int64_t)ox * nO + oy) * nV + box_lo(pbx) + rr) * nV + box_lo(qbx) + cc] : 0.0;
    }
    for (int e = tid; e < 3 * BX * 3; e += THREADS) {
      const int bxi = e / (BX * 3), rr = (e / 3) % BX, z = e % 3;
      const int32_t oz = z == 0 ? K : (z == 1 ? J : I);
      t1s[e] = rr < box_ex(bxi) ? p.T1[(int64_t)(box_lo(bxi) + rr) * nO + oz] : 0.0;
    }
    for (int e = tid; e < 3 * BX; e += THREADS) {
      const int bxi = e / BX, rr = e % BX;
      epv[e] = rr < box_ex(bxi) ? p.eps_v[box_lo(bxi) + rr] : 0.0;
    }
  }
  compute_sync();
  double s = 0.0;
  const double dijk = p.eps_o[I] + p.eps_o[J] + p.eps_o[K];
  for (int idx = tid; idx < BX * BX * BX; idx += THREADS) {
    const int la = idx / (BX * BX), lb = (idx / BX) % BX, lc = idx % BX;
    if (la >= ex[0] || lb >= ex[1] || lc >= ex[2]) continue;
    const int32_t a = lo[0] + la, b = lo[1] + lb, c = lo[2] + lc;
    if (!(a < b && b < c)) continue;
    const double W = cube[cidx(la, lb, lc)];
    // V1 (Eq. tensort2): pairs (x,y;z) = (i,j;k)+, (i,k;j)-, (j,k;i)+  x  (p,q;r) = (a,b;c)+, (a,c;b)-, (b,c;a)+
    double v1 = 0.0;
#pragma unroll
    for (int pr = 0; pr < 3; ++pr) {
      const double* vt = vds + pr * 3 * BX * VDP;
      const double inner = vt[(0 * BX + la) * VDP + lb] * t1s[(2 * BX + lc) * 3 + pr]
                         - vt[(1 * BX + la) * VDP + lc] * t1s[(1 * BX + lb) * 3 + pr]
                         + vt[(2 * BX + lb) * VDP + lc] * t1s[(0 * BX + la) * 3 + pr];
      v1 = (pr == 1) ? v1 - inner : v1 + inner;
    }
    const double D = dijk - epv[la] - epv[BX + lb] - epv[2 * BX + lc];
    s += (W + v1) * W / D;
  }
  red[tid] = s;
  compute_sync();
  for (int o = THREADS / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    compute_sync();
  }
  if (tid == 0) p.partials[u] = red[0];
}

// -------------------------------------------------------------------------------------------------
// Pair variant (opt-in, TT_TRIPLES_PAIR=1; measured slower at O=40 V=200: 4.59 s vs 3.37 s -- one
// 16-warp CTA per SM with 3 stages of 44 KB hides the TMA latency worse than two 8-warp CTAs): one CTA computes TWO units with the same box triple and occupied
// triples (i,j,k1), (i,j,k2).  In every segment of the K loop one of the two operands is the same for
// both triples -- the Q tile (depends on one occupied index) in the segments (A,s=1), (A,s=2), (B,s=0),
// (B,s=1), the P tile (depends on the pair) in (A,s=0), (B,s=2) -- so that operand is loaded once: 2/3
// of the K range moves one Q tile for two triples.  Warps 0-7 compute the first triple, 8-15 the second;
// each triple keeps its own cube and partial, so the energies are bitwise those of the single kernel.
namespace {
constexpr int PTHREADS = 2 * THREADS;
constexpr int PNS = 3;
constexpr int PSTAGE = 2 * TP_BYTES + 2 * TQ_BYTES;   // P1 P2 Q1 Q2
}  // namespace

__global__ void __launch_bounds__(PTHREADS, 1)
    triples_pair_tma_kernel(const TriplesParams p, const __grid_constant__ CUtensorMap mVO,
                            const __grid_constant__ CUtensorMap mT2P, const __grid_constant__ CUtensorMap mT2Q,
                            const __grid_constant__ CUtensorMap mVV) {
  extern __shared__ __align__(128) unsigned char psm_raw[];
  unsigned char* base = psm_raw + ((128 - ((unsigned)__cvta_generic_to_shared(psm_raw) & 127)) & 127);   // stays in the shared window (LDS, not generic LD)
  double* cubes = reinterpret_cast<double*>(base + PNS * PSTAGE);   // [2][BX^3]
  double* red = cubes + 2 * BX * BX * BX;                          // [PTHREADS]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + PTHREADS);    // [PNS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = warp >> 3, lw = warp & 7;                          // triple of this warp, warp inside it
  const int2 pr = p.pairs[blockIdx.x];
  const int64_t u1 = pr.x;
  const bool two = pr.y == 2;
  const int2 un1 = p.units[u1];
  const int4 bx = p.box3[un1.x];
  const int4 tr1 = p.trip[un1.y];
  const int4 tr2 = two ? p.trip[p.units[u1 + 1].y] : tr1;
  const int32_t nO = p.nO, nV = p.nV;
  const int32_t lo[3] = {p.box_lo[bx.x], p.box_lo[bx.y], p.box_lo[bx.z]};
  const int32_t ex[3] = {p.box_ext[bx.x], p.box_ext[bx.y], p.box_ext[bx.z]};
  const int32_t I = tr1.x, J = tr1.y, K1 = tr1.z, K2 = tr2.z;
  const int32_t sA = (nO + KC - 1) / KC, sB = (nV + KC - 1) / KC;
  const int32_t nst = 3 * sA + 3 * sB;
  const int32_t total = 3 * nst;
  double* cube = cubes + h * BX * BX * BX;
  if (tid == 0) {
    for (int q = 0; q < PNS; ++q) tbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mVO) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mT2P) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mT2Q) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mVV) : "memory");
  }
  __syncthreads();
  // segment sharing: 0 = (A,s=0) P shared; 1,2 = (A,s=1/2) Q shared; 3,4 = (B,s=0/1) Q shared; 5 = (B,s=2) P shared
  auto issue = [&](int32_t t) {
    const int g = t / nst;
    int32_t r = t - g * nst;
    const int32_t lo_r = g == 0 ? lo[0] : (g == 1 ? lo[1] : lo[2]);
    const int32_t lo_p = g == 0 ? lo[1] : lo[0];
    const int32_t lo_q = g == 2 ? lo[1] : lo[2];
    unsigned char* st = base + (t % PNS) * PSTAGE;
    double* P1 = reinterpret_cast<double*>(st);
    double* P2 = reinterpret_cast<double*>(st + TP_BYTES);
    double* Q1 = reinterpret_cast<double*>(st + 2 * TP_BYTES);
    double* Q2 = reinterpret_cast<double*>(st + 2 * TP_BYTES + TQ_BYTES);
    uint64_t* bar = &full[t % PNS];
    if (r < 3 * sA) {
      const int s = r / sA;
      const int32_t m0 = (r - s * sA) * KC;
      if (s == 0) {          // P = VO[I][J] shared, Q = T2[m][k] per triple
        tbar_expect(bar, (unsigned)(TP_BYTES + (two ? 2 : 1) * TQ_BYTES));
        tma4(P1, &mVO, lo_r, m0, J, I, bar);
        tma4(Q1, &mT2Q, lo_q, lo_p, K1, m0, bar);
        if (two) tma4(Q2, &mT2Q, lo_q, lo_p, K2, m0, bar);
      } else {               // s=1: P = VO[I][k], Q = T2[m][J];  s=2: P = VO[J][k], Q = T2[m][I]
        const int32_t x = (s == 2) ? J : I, z = (s == 1) ? J : I;
        tbar_expect(bar, (unsigned)((two ? 2 : 1) * TP_BYTES + TQ_BYTES));
        tma4(P1, &mVO, lo_r, m0, K1, x, bar);
        if (two) tma4(P2, &mVO, lo_r, m0, K2, x, bar);
        tma4(Q1, &mT2Q, lo_q, lo_p, z, m0, bar);
      }
    } else {
      r -= 3 * sA;
      const int s = r / sB;
      const int32_t e0 = (r - s * sB) * KC;
      if (s == 2) {          // P = T2[I][J][e] shared, Q = VV[e][k] per triple
        tbar_expect(bar, (unsigned)(TP_BYTES + (two ? 2 : 1) * TQ_BYTES));
        tma4(P1, &mT2P, lo_r, e0, J, I, bar);
        tma4(Q1, &mVV, lo_q, lo_p, K1, e0, bar);
        if (two) tma4(Q2, &mVV, lo_q, lo_p, K2, e0, bar);
      } else {               // s=0: P = T2[J][k][e], Q = VV[e][I];  s=1: P = T2[I][k][e], Q = VV[e][J]
        const int32_t y = (s == 0) ? J : I, x = (s == 0) ? I : J;
        tbar_expect(bar, (unsigned)((two ? 2 : 1) * TP_BYTES + TQ_BYTES));
        tma4(P1, &mT2P, lo_r, e0, K1, y, bar);
        if (two) tma4(P2, &mT2P, lo_r, e0, K2, y, bar);
        tma4(Q1, &mVV, lo_q, lo_p, x, e0, bar);
      }
    }
  };
  if (tid == 0)
    for (int t = 0; t < PNS && t < total; ++t) issue(t);

  double acc[2][NFR][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int f = 0; f < NFR; ++f) acc[a][f][0] = acc[a][f][1] = 0.0;
  const bool active = h == 0 || two;
  int g = 0, sg = 0, slot = 0;
  unsigned phase = 0;
#pragma unroll 1
  for (int t = 0; t < total; ++t) {
    tbar_wait(&full[slot], phase);
    const int seg = sg < 3 * sA ? sg / sA : 3 + (sg - 3 * sA) / sB;
    const bool pshared = seg == 0 || seg == 5;
    const unsigned char* st = base + slot * PSTAGE;
    const double* P = reinterpret_cast<const double*>(st + ((h && !pshared) ? TP_BYTES : 0));
    const double* Q = reinterpret_cast<const double*>(st + 2 * TP_BYTES + ((h && pshared) ? TQ_BYTES : 0));
    const bool neg = seg < 3 ? seg == 1 : seg != 4;   // m sums (+,-,+), e sums (-,+,-)
    const long long sgm = neg ? (long long)0x8000000000000000ull : 0ll;
    if (active) {
#pragma unroll
      for (int kk = 0; kk < KC / 4; ++kk) {
        const int kl = kk * 4 + (lane & 3);
        const double a0 = __longlong_as_double(__double_as_longlong(P[kl * TPW + (lane >> 2)]) ^ sgm);
        const double a1 = __longlong_as_double(__double_as_longlong(P[kl * TPW + 8 + (lane >> 2)]) ^ sgm);
#pragma unroll
        for (int f = 0; f < NFR; ++f) {
          const int col = lw * CW + f * 8 + (lane >> 2);
          const double b = Q[kl * TQS + (col / BX) * TQW + (col % BX)];
          dmma(acc[0][f], a0, b);
          dmma(acc[1][f], a1, b);
        }
      }
    }
    __syncthreads();
    if (tid == 0 && t + PNS < total) issue(t + PNS);
    slot = (slot + 1 == PNS) ? 0 : slot + 1;
    if (slot == 0) phase ^= 1;
    if (++sg == nst) {
#pragma unroll
      for (int rf = 0; rf < 2; ++rf)
#pragma unroll
        for (int f = 0; f < NFR; ++f)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int row = rf * 8 + (lane >> 2);
            const int col = lw * CW + f * 8 + 2 * (lane & 3) + hh;
            const int pp = col / BX, q = col % BX;
            const double v = acc[rf][f][hh];
            if (g == 0) cube[cidx(row, pp, q)] = v;
            else if (g == 1) cube[cidx(pp, row, q)] -= v;
            else cube[cidx(pp, q, row)] += v;
            acc[rf][f][hh] = 0.0;
          }
      __syncthreads();
      sg = 0;
      ++g;
    }
  }
  // Eq. cc14 over each triple's cube (threads 256 h .. 256 h + 255), one partial per unit
  const int ht = tid & (THREADS - 1);
  const int32_t Kh = h ? K2 : K1;
  double s = 0.0;
  if (active) {
    const double dijk = p.eps_o[I] + p.eps_o[J] + p.eps_o[Kh];
    for (int idx = ht; idx < BX * BX * BX; idx += THREADS) {
      const int la = idx / (BX * BX), lb = (idx / BX) % BX, lc = idx % BX;
      if (la >= ex[0] || lb >= ex[1] || lc >= ex[2]) continue;
      const int32_t a = lo[0] + la, b = lo[1] + lb, c = lo[2] + lc;
      if (!(a < b && b < c)) continue;
      const double W = cube[cidx(la, lb, lc)];
      double v1 = 0.0;
      const int32_t ox[3] = {I, I, J}, oy[3] = {J, Kh, Kh}, oz[3] = {Kh, J, I};
      const int32_t vp[3] = {a, a, b}, vq[3] = {b, c, c}, vr[3] = {c, b, a};
#pragma unroll
      for (int q3 = 0; q3 < 3; ++q3) {
        double inner = 0.0;
#pragma unroll
        for (int pq = 0; pq < 3; ++pq) {
          const double term = p.VD[(((int64_t)ox[q3] * nO + oy[q3]) * nV + vp[pq]) * nV + vq[pq]] *
                              p.T1[(int64_t)vr[pq] * nO + oz[q3]];
          inner = (pq == 1) ? inner - term : inner + term;
        }
        v1 = (q3 == 1) ? v1 - inner : v1 + inner;
      }
      const double D = dijk - p.eps_v[a] - p.eps_v[b] - p.eps_v[c];
      s += (W + v1) * W / D;
    }
  }
  red[tid] = s;
  __syncthreads();
  for (int o = THREADS / 2; o > 0; o >>= 1) {
    if (ht < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (ht == 0 && active) p.partials[u1 + h] = red[tid];
}

// -------------------------------------------------------------------------------------------------
// Cluster variant (opt-in, TT_TRIPLES_CLUSTER=1; measured slower: 5.79 s vs 3.08 s at O=40 V=200 --
// both CTAs must release a slot before either refills it, so each CTA runs at the pace of the other's
// slowest warp through only 3 slots): a 2-CTA thread-block cluster computes the two units (i,j,k1), (i,j,k2) of
// a pair (same box triple, same spin of k: identical segment ranges).  In every segment one operand is
// the same for both triples (the pair analysis above); CTA 0 loads it ONCE with a TMA multicast into
// both CTAs' shared memory, and each CTA loads its own per-triple operand.  L2->SM traffic per stage
// drops from P + Q to about (P + Q/2) or (P/2 + Q): ~1/3 less, while each CTA keeps the single-unit
// layout (8 compute warps + producer warp, 2 CTAs per SM).  Each slot's "empty" barrier collects the
// releases of BOTH CTAs' compute warps (local arrive + remote arrive on the peer through its cluster
// address), so neither producer refills a slot the other CTA still reads or the multicast still
// targets.  A lone unit (odd run of k) gives both CTAs the same unit; CTA 1 then writes no partial.
size_t triples_cluster_smem();

namespace {
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tbar_arrive_peer(uint64_t* bar, unsigned peer) {
  unsigned s = (unsigned)__cvta_generic_to_shared(bar), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(s), "r"(peer));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(r) : "memory");
}
__device__ __forceinline__ void tma4_mc(void* smem, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar,
                                        unsigned short mask) {
  unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;\n"
      ::"r"(d), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b), "h"(mask)
      : "memory");
}
}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TTHREADS, 2)
    triples_cluster_tma_kernel(const TriplesParams p, const __grid_constant__ CUtensorMap mVO,
                               const __grid_constant__ CUtensorMap mT2P, const __grid_constant__ CUtensorMap mT2Q,
                               const __grid_constant__ CUtensorMap mVV) {
  extern __shared__ __align__(128) unsigned char csm_raw[];
  unsigned char* base = csm_raw + ((128 - ((unsigned)__cvta_generic_to_shared(csm_raw) & 127)) & 127);   // stays in the shared window (LDS, not generic LD)
  double* cube = reinterpret_cast<double*>(base + TNS * TSTAGE);   // [BX][BX][BX]
  double* red = cube + BX * BX * BX;                               // [THREADS]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + THREADS);     // [TNS]
  uint64_t* empty = full + TNS;                                    // [TNS]
  int32_t* segb = reinterpret_cast<int32_t*>(empty + TNS);         // [3][6]
  int32_t* segn = segb + 18;                                       // [3][6]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned crank = cluster_rank(), peer = crank ^ 1u;
  const int2 pr = p.pairs[blockIdx.x >> 1];
  const bool two = pr.y == 2;
  const int64_t u = (int64_t)pr.x + ((two && crank) ? 1 : 0);
  const int2 un = p.units[u];
  const int4 bx = p.box3[un.x];
  const int4 tr = p.trip[un.y];
  const int32_t nO = p.nO, nV = p.nV;
  const int32_t lo[3] = {p.box_lo[bx.x], p.box_lo[bx.y], p.box_lo[bx.z]};
  const int32_t ex[3] = {p.box_ext[bx.x], p.box_ext[bx.y], p.box_ext[bx.z]};
  const int32_t I = tr.x, J = tr.y, K = tr.z;
  if (tid == 0) {
    for (int q = 0; q < TNS; ++q) {
      tbar_init(&full[q], 1);
      tbar_init(&empty[q], 2 * NWARP);   // this CTA's and the peer's compute warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < 18) {   // segment ranges (identical in both CTAs: same i, j and spin of k)
    const int g = tid / 6, sg = tid % 6;
    const int32_t oh = p.o_half, vh = p.v_half;
    auto so = [&](int32_t x) { return oh ? (x < oh ? 1 : -1) : 0; };
    auto sv = [&](int32_t v) { return vh ? (v < vh ? 1 : -1) : 0; };
    const int32_t sr = sv(g == 0 ? lo[0] : (g == 1 ? lo[1] : lo[2]));
    const int32_t sp = sv(g == 0 ? lo[1] : lo[0]), sq = sv(g == 2 ? lo[1] : lo[2]);
    int32_t b = 0, e = 0;
    if (sg < 3) {
      const int32_t x = (sg == 2) ? J : I, y = (sg == 0) ? J : K;
      const int32_t sm = so(x) + so(y) - sr;
      if (!oh) { b = 0; e = nO; }
      else if (sm == 1) { b = 0; e = oh; }
      else if (sm == -1) { b = oh; e = nO; }
    } else {
      const int32_t x = (sg == 3) ? I : (sg == 4 ? J : K);
      const int32_t se = sp + sq - so(x);
      if (!vh) { b = 0; e = nV; }
      else if (se == 1) { b = 0; e = vh; }
      else if (se == -1) { b = vh; e = nV; }
    }
    segb[tid] = b;
    segn[tid] = (e - b + KC - 1) / KC;
  }
  __syncthreads();
  cluster_sync_all();   // the peer's barriers are initialised before any multicast or remote arrive

  if (warp == NWARP) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mVO) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mT2P) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mT2Q) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mVV) : "memory");
      int slot = 0;
      unsigned phase = 1;
      for (int g = 0; g < 3; ++g) {
        const int32_t lo_r = g == 0 ? lo[0] : (g == 1 ? lo[1] : lo[2]);
        const int32_t lo_p = g == 0 ? lo[1] : lo[0];
        const int32_t lo_q = g == 2 ? lo[1] : lo[2];
        for (int sg = 0; sg < 6; ++sg) {
          const int32_t n = segn[g * 6 + sg];
          // shared operand of the segment: P in (m, s=0) and (e, s=2), else Q
          const bool pshared = sg == 0 || sg == 5;
          for (int jj = 0; jj < n; ++jj) {
            const int32_t k0 = segb[g * 6 + sg] + jj * KC;
            tbar_wait(&empty[slot], phase);
            unsigned char* st = base + slot * TSTAGE;
            double* P = reinterpret_cast<double*>(st);
            double* Q = reinterpret_cast<double*>(st + TP_BYTES);
            tbar_expect(&full[slot], (unsigned)TSTAGE);   // own operand + the multicast one
            if (sg < 3) {
              const int32_t x = (sg == 2) ? J : I, y = (sg == 0) ? J : K, z = (sg == 0) ? K : (sg == 1 ? J : I);
              if (pshared) {
                if (crank == 0) tma4_mc(P, &mVO, lo_r, k0, y, x, &full[slot], 3);
                tma4(Q, &mT2Q, lo_q, lo_p, z, k0, &full[slot]);
              } else {
                tma4(P, &mVO, lo_r, k0, y, x, &full[slot]);
                if (crank == 0) tma4_mc(Q, &mT2Q, lo_q, lo_p, z, k0, &full[slot], 3);
              }
            } else {
              const int s3 = sg - 3;
              const int32_t x = (s3 == 0) ? I : (s3 == 1 ? J : K), y = (s3 == 0) ? J : I, z = (s3 == 2) ? J : K;
              if (pshared) {
                if (crank == 0) tma4_mc(P, &mT2P, lo_r, k0, z, y, &full[slot], 3);
                tma4(Q, &mVV, lo_q, lo_p, x, k0, &full[slot]);
              } else {
                tma4(P, &mT2P, lo_r, k0, z, y, &full[slot]);
                if (crank == 0) tma4_mc(Q, &mVV, lo_q, lo_p, x, k0, &full[slot], 3);
              }
            }
            if (++slot == TNS) { slot = 0; phase ^= 1; }
          }
        }
      }
    }
    __syncwarp();
    cluster_sync_all();
    return;
  }

  // ------------------------------------------------------------------ compute warps (8)
  double acc[2][NFR][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int f = 0; f < NFR; ++f) acc[a][f][0] = acc[a][f][1] = 0.0;
  int slot = 0;
  unsigned phase = 0;
#pragma unroll 1
  for (int g = 0; g < 3; ++g) {
    uint32_t need = 0;
#pragma unroll
    for (int rf = 0; rf < 2; ++rf)
#pragma unroll
      for (int f = 0; f < NFR; ++f) {
        const int col = warp * CW + f * 8;
        if (frag_needed(g, 8 * rf, col / BX, col % BX, lo, ex)) need |= 1u << (rf * NFR + f);
      }
#pragma unroll 1
    for (int sg = 0; sg < 6; ++sg) {
      const int32_t n = segn[g * 6 + sg];
      const bool neg = sg < 3 ? sg == 1 : sg != 4;
      const long long sgm = neg ? (long long)0x8000000000000000ull : 0ll;
#pragma unroll 1
      for (int jj = 0; jj < n; ++jj) {
        tbar_wait(&full[slot], phase);
        if (need) {
          const double* P = reinterpret_cast<const double*>(base + slot * TSTAGE);
          const double* Q = reinterpret_cast<const double*>(base + slot * TSTAGE + TP_BYTES);
#pragma unroll
          for (int kk = 0; kk < KC / 4; ++kk) {
            const int kl = kk * 4 + (lane & 3);
            const double a0 = __longlong_as_double(__double_as_longlong(P[kl * TPW + (lane >> 2)]) ^ sgm);
            const double a1 = __longlong_as_double(__double_as_longlong(P[kl * TPW + 8 + (lane >> 2)]) ^ sgm);
#pragma unroll
            for (int f = 0; f < NFR; ++f) {
              const int col = warp * CW + f * 8 + (lane >> 2);
              const double b = Q[kl * TQS + (col / BX) * TQW + (col % BX)];
              if (need & (1u << f)) dmma(acc[0][f], a0, b);
              if (need & (1u << (NFR + f))) dmma(acc[1][f], a1, b);
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          tbar_arrive(&empty[slot]);
          tbar_arrive_peer(&empty[slot], peer);
        }
        if (++slot == TNS) { slot = 0; phase ^= 1; }
      }
    }
#pragma unroll
    for (int rf = 0; rf < 2; ++rf)
#pragma unroll
      for (int f = 0; f < NFR; ++f)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = rf * 8 + (lane >> 2);
          const int col = warp * CW + f * 8 + 2 * (lane & 3) + h;
          const int pp = col / BX, q = col % BX;
          const double v = acc[rf][f][h];
          if (g == 0) cube[cidx(row, pp, q)] = v;
          else if (g == 1) cube[cidx(pp, row, q)] -= v;
          else cube[cidx(pp, q, row)] += v;
          acc[rf][f][h] = 0.0;
        }
    compute_sync();
  }
  double s = 0.0;
  const double dijk = p.eps_o[I] + p.eps_o[J] + p.eps_o[K];
  for (int idx = tid; idx < BX * BX * BX; idx += THREADS) {
    const int la = idx / (BX * BX), lb = (idx / BX) % BX, lc = idx % BX;
    if (la >= ex[0] || lb >= ex[1] || lc >= ex[2]) continue;
    const int32_t a = lo[0] + la, b = lo[1] + lb, c = lo[2] + lc;
    if (!(a < b && b < c)) continue;
    const double W = cube[cidx(la, lb, lc)];
    double v1 = 0.0;
    const int32_t ox[3] = {I, I, J}, oy[3] = {J, K, K}, oz[3] = {K, J, I};
    const int32_t vp[3] = {a, a, b}, vq[3] = {b, c, c}, vr[3] = {c, b, a};
#pragma unroll
    for (int q3 = 0; q3 < 3; ++q3) {
      double inner = 0.0;
#pragma unroll
      for (int pq = 0; pq < 3; ++pq) {
        const double term = p.VD[(((int64_t)ox[q3] * nO + oy[q3]) * nV + vp[pq]) * nV + vq[pq]] *
                            p.T1[(int64_t)vr[pq] * nO + oz[q3]];
        inner = (pq == 1) ? inner - term : inner + term;
      }
      v1 = (q3 == 1) ? v1 - inner : v1 + inner;
    }
    const double D = dijk - p.eps_v[a] - p.eps_v[b] - p.eps_v[c];
    s += (W + v1) * W / D;
  }
  red[tid] = s;
  compute_sync();
  for (int o = THREADS / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    compute_sync();
  }
  if (tid == 0 && (two || crank == 0)) p.partials[u] = red[0];
  cluster_sync_all();   // no CTA leaves while its peer may still arrive on its barriers
}

cudaError_t launch_triples_cluster(const TriplesParams& p, const void* maps, int64_t npairs, cudaStream_t s) {
  if (npairs <= 0) return cudaSuccess;
  static bool attr = false;
  const size_t smem = triples_cluster_smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(triples_cluster_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const CUtensorMap* m = static_cast<const CUtensorMap*>(maps);
  triples_cluster_tma_kernel<<<(unsigned)(2 * npairs), TTHREADS, smem, s>>>(p, m[0], m[1], m[2], m[3]);
  return cudaGetLastError();
}

size_t triples_pair_smem() {
  return 128 + (size_t)PNS * PSTAGE + sizeof(double) * (2 * BX * BX * BX + PTHREADS) + 8 * PNS;
}

cudaError_t launch_triples_pair(const TriplesParams& p, const void* maps, int64_t npairs, cudaStream_t s) {
  if (npairs <= 0) return cudaSuccess;
  static bool attr = false;
  const size_t smem = triples_pair_smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(triples_pair_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const CUtensorMap* m = static_cast<const CUtensorMap*>(maps);
  triples_pair_tma_kernel<<<(unsigned)npairs, PTHREADS, smem, s>>>(p, m[0], m[1], m[2], m[3]);
  return cudaGetLastError();
}

size_t triples_cluster_smem() {   // padded-layout TMA stages (cluster variant)
  return 128 + (size_t)TNS * TSTAGE + sizeof(double) * (BX * BX * BX + THREADS) + 16 * TNS + 4 * 36;
}
size_t triples_tma_smem() {   // the default kernel (bulk-copy stages)
  return 128 + (size_t)BNS * BSTAGE + sizeof(double) * (BX * BX * BX + THREADS) + 16 * BNS + 4 * 36;
}

cudaError_t launch_triples_tma(const TriplesParams& p, int64_t nunits, cudaStream_t s) {
  if (nunits <= 0) return cudaSuccess;
  static bool attr = false;
  const size_t smem = triples_tma_smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(triples_fused_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  triples_fused_tma_kernel<<<(unsigned)nunits, TTHREADS, smem, s>>>(p);
  return cudaGetLastError();
}

size_t triples_fused_smem() {
  return sizeof(double) * ((size_t)NS * KC * (PS + QS) + BX * BX * BX + THREADS);
}

cudaError_t launch_retile(const RetileParams& p, int64_t nseg, cudaStream_t s) {
  if (nseg <= 0) return cudaSuccess;
  retile_kernel<<<(unsigned)nseg, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_triples_fused(const TriplesParams& p, int64_t nunits, cudaStream_t s) {
  if (nunits <= 0) return cudaSuccess;
  static bool attr = false;
  const size_t smem = triples_fused_smem();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(triples_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  triples_fused_kernel<<<(unsigned)nunits, THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tt
