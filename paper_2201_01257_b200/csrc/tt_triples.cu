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
