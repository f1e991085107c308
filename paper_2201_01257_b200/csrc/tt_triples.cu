// tt_triples.cu -- sm_100a kernels of the perturbative-triples path (PAPER Eqs. cc14,
// tensort, tensort2, P343-413) that are not contractions: re-tiling copies of the inputs (the summed
// labels m, e are staged on one tile per spin range so each of the 18 Eq. tensort terms is a single
// K = O or K = V pass of the DMMA kernel), and the fused energy assembly of Eq. cc14.
#include "tt_launch.h"

namespace tt {

// dst block element e -> global coordinates -> the src block (another tiling of the same index spaces)
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
      const int32_t t = p.g2t[q][g[q]];
      const int64_t o0 = p.toff[q][t];
      bid = bid * p.sgrid[q] + t;
      el = el * (p.toff[q][t + 1] - o0) + (g[q] - o0);
    }
    const int64_t so = p.sblk_off[bid];
    dst[e] = so >= 0 ? p.src[so + el] : 0.0;
  }
}

// Eq. cc14 over one chunk of one W block: sum over a<b<c, i<j<k of (W + V1) * W / D, V1 = Eq. tensort2
// (nine Voovv * T1 products read from their blocks), D from the orbital energies.  One partial per CTA
// (fixed thread order + fixed tree: deterministic, reading R12).
__global__ void triples_energy_kernel(const TriplesParams p) {
  __shared__ double red[256];
  const Segment sg = p.segs[blockIdx.x];
  const TriplesBlk& B = p.blks[sg.desc];
  const double* w = p.W + B.w_off;
  const int32_t ea = B.ext[0], eb = B.ext[1], ec = B.ext[2], ei = B.ext[3], ej = B.ext[4], ek = B.ext[5];
  const int32_t le[6] = {ea, eb, ec, ei, ej, ek};
  double s = 0.0;
  for (int64_t e = sg.e0 + threadIdx.x; e < sg.e1; e += blockDim.x) {
    int64_t r = e;
    int32_t l[6];
    for (int q = 5; q >= 0; --q) { l[q] = (int32_t)(r % le[q]); r /= le[q]; }
    const int32_t a = B.org[0] + l[0], b = B.org[1] + l[1], c = B.org[2] + l[2];
    const int32_t i = B.org[3] + l[3], j = B.org[4] + l[4], k = B.org[5] + l[5];
    if (!(a < b && b < c && i < j && j < k)) continue;
    const double W = w[e];
    // V1: pairs (x,y) = (i,j) z=k +, (i,k) z=j -, (j,k) z=i +; (p,q) = (a,b) r=c +, (a,c) r=b -, (b,c) r=a +
    const int32_t lo[3][3] = {{l[3], l[4], l[5]}, {l[3], l[5], l[4]}, {l[4], l[5], l[3]}};
    const int32_t eo[3][3] = {{ei, ej, ek}, {ei, ek, ej}, {ej, ek, ei}};
    const int32_t lv[3][3] = {{l[0], l[1], l[2]}, {l[0], l[2], l[1]}, {l[1], l[2], l[0]}};
    const int32_t ev[3][3] = {{ea, eb, ec}, {ea, ec, eb}, {eb, ec, ea}};
    double v1 = 0.0;
#pragma unroll
    for (int pr = 0; pr < 3; ++pr) {
      double inner = 0.0;
#pragma unroll
      for (int pq = 0; pq < 3; ++pq) {
        const int64_t vo = B.v_off[pr * 3 + pq], to = B.t_off[pr * 3 + pq];
        if (vo < 0 || to < 0) continue;
        const int64_t vi = (((int64_t)lo[pr][0] * eo[pr][1] + lo[pr][1]) * ev[pq][0] + lv[pq][0]) * ev[pq][1] + lv[pq][1];
        const int64_t ti = (int64_t)lv[pq][2] * eo[pr][2] + lo[pr][2];
        const double term = p.Voovv[vo + vi] * p.T1[to + ti];
        inner = (pq == 1) ? inner - term : inner + term;
      }
      v1 = (pr == 1) ? v1 - inner : v1 + inner;
    }
    const double D = p.eps_o[i] + p.eps_o[j] + p.eps_o[k] - p.eps_v[a] - p.eps_v[b] - p.eps_v[c];
    s += (W + v1) * W / D;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) p.partials[blockIdx.x] = red[0];
}

cudaError_t launch_retile(const RetileParams& p, int64_t nseg, cudaStream_t s) {
  if (nseg <= 0) return cudaSuccess;
  retile_kernel<<<(unsigned)nseg, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_triples_energy(const TriplesParams& p, int64_t nseg, cudaStream_t s) {
  if (nseg <= 0) return cudaSuccess;
  triples_energy_kernel<<<(unsigned)nseg, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tt
