/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct FP64 loops that define what
 * the B200 path must compute.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code with paper_2201_01257_b200/.
 *
 * Operations follow PAPER.md §3.1 (P172-174, grammar rules 5-7):
 *   set          A(i,l)  = alpha                                   (P172)
 *   add          A(i,l) += alpha * D(l,i)   (label permutation)    (P173)
 *   contraction  C(i,a) += alpha * A(i,l) * B(l,a)                 (P174)
 * with the general beta of BASELINE.json north_star:  C <- beta*C + alpha*op  (beta = 0 for "=",
 * C then never read; reading R3/R4).
 *
 * Summation order (reading R12): for every output element, the contracted index tuple is
 * walked row-major with contracted labels in order of first appearance in A, and the products are
 * added one at a time in that order, starting from 0.0.  Built with -O2 -ffp-contract=off and no
 * fast-math so that every product is rounded before it is added (IEEE round-to-nearest).
 */
#include <stdint.h>
#include <stddef.h>

#define MAXL 16

/* Naive strided contraction over dense global arrays.
 *   free labels (C order): ext_f[nf], stride in C / A / B (0 where the label is absent from A or B)
 *   contracted labels (order of first appearance in A): ext_k[nk], stride in A / B
 *   cmask: dense u8 over C (1 = element lies in a non-zero C block); NULL = all ones.
 * C[x] <- beta*C[x] + alpha*sum   on masked elements; beta == 0 => C[x] is not read. */
void orc_contract_naive(int nf, const int64_t* ext_f, const int64_t* sfc, const int64_t* sfa,
                        const int64_t* sfb, int nk, const int64_t* ext_k, const int64_t* ska,
                        const int64_t* skb, double* C, const double* A, const double* B,
                        const uint8_t* cmask, double alpha, double beta) {
  int64_t fi[MAXL], ki[MAXL];
  for (int d = 0; d < nf; ++d) { fi[d] = 0; if (ext_f[d] == 0) return; }
  for (;;) {
    int64_t oc = 0, oa = 0, ob = 0;
    for (int d = 0; d < nf; ++d) { oc += fi[d] * sfc[d]; oa += fi[d] * sfa[d]; ob += fi[d] * sfb[d]; }
    if (cmask == NULL || cmask[oc]) {
      double s = 0.0;
      int empty = 0;
      for (int d = 0; d < nk; ++d) { ki[d] = 0; if (ext_k[d] == 0) empty = 1; }
      if (!empty) {
        for (;;) {
          int64_t ia = oa, ib = ob;
          for (int d = 0; d < nk; ++d) { ia += ki[d] * ska[d]; ib += ki[d] * skb[d]; }
          double p = A[ia] * B[ib];
          s = s + p;
          int d = nk - 1;
          while (d >= 0) { if (++ki[d] < ext_k[d]) break; ki[d] = 0; --d; }
          if (d < 0) break;
        }
      }
      double as = alpha * s;
      C[oc] = (beta == 0.0) ? as : beta * C[oc] + as;
    }
    int d = nf - 1;
    while (d >= 0) { if (++fi[d] < ext_f[d]) break; fi[d] = 0; --d; }
    if (d < 0) break;
  }
}

/* Same sums, operands pre-gathered (memory order only) into A2[fa][K], B2[fb][K] with the
 * contracted tuple in the same row-major order as orc_contract_naive:
 *   P[fa*nfb + fb] = sum_k A2[fa*K + k] * B2[fb*K + k]   (sequential in k).
 * Bit-identical to the naive loop (tests check this). OpenMP over output rows only. */
void orc_contract_gathered(int64_t nfa, int64_t nfb, int64_t K, const double* A2, const double* B2,
                           double* P) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t fa = 0; fa < nfa; ++fa) {
    const double* a = A2 + fa * K;
    for (int64_t fb = 0; fb < nfb; ++fb) {
      const double* b = B2 + fb * K;
      double s = 0.0;
      for (int64_t k = 0; k < K; ++k) { double p = a[k] * b[k]; s = s + p; }
      P[fa * nfb + fb] = s;
    }
  }
}

/* Sequential dot product s = sum_i a[i]*b[i] (scalar contraction, sampled elements). */
double orc_dot(int64_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) { double p = a[i] * b[i]; s = s + p; }
  return s;
}

/* Many independent sequential dots: out[r] = sum_k a[r*K+k]*b[r*K+k]. */
void orc_dots(int64_t nrows, int64_t K, const double* a, const double* b, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nrows; ++r) out[r] = orc_dot(K, a + r * K, b + r * K);
}

/* Freivalds projection of one output block:
 *   y[m] = sum_n Cblk[m*N+n] x[n]        and       z[m] = sum_p sum_k Ap[m*K+k] (sum_n Bp[k*N+n] x[n])
 * Here only the plain matrix-vector product y = M x (row-major M rows x cols) is provided. */
void orc_matvec(int64_t rows, int64_t cols, const double* M, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0.0;
    for (int64_t c = 0; c < cols; ++c) { double p = M[r * cols + c] * x[c]; s = s + p; }
    y[r] = s;
  }
}

/* Naive three-operand contraction (PAPER Eq. cc9, P293-300: the unfactorized n_o^4 n_u^4 loop):
 *   C[x] <- beta*C[x] + alpha * sum_{y} (A[.] * B[.]) * D[.]
 * free labels (C order) ext_f[nf] with strides in C/A/B/D (0 = absent); summed labels (every label
 * not in C, order of first appearance in A, then B, then D) ext_k[nk] with strides in A/B/D.
 * Sequential sum per output element, row-major over the summed tuple.  cmask as orc_contract_naive. */
void orc_contract3_naive(int nf, const int64_t* ext_f, const int64_t* sfc, const int64_t* sfa,
                         const int64_t* sfb, const int64_t* sfd, int nk, const int64_t* ext_k,
                         const int64_t* ska, const int64_t* skb, const int64_t* skd, double* C,
                         const double* A, const double* B, const double* D, const uint8_t* cmask,
                         double alpha, double beta) {
  int64_t fi[MAXL], ki[MAXL];
  for (int d = 0; d < nf; ++d) { fi[d] = 0; if (ext_f[d] == 0) return; }
  for (;;) {
    int64_t oc = 0, oa = 0, ob = 0, od = 0;
    for (int d = 0; d < nf; ++d) {
      oc += fi[d] * sfc[d]; oa += fi[d] * sfa[d]; ob += fi[d] * sfb[d]; od += fi[d] * sfd[d];
    }
    if (cmask == NULL || cmask[oc]) {
      double s = 0.0;
      int empty = 0;
      for (int d = 0; d < nk; ++d) { ki[d] = 0; if (ext_k[d] == 0) empty = 1; }
      if (!empty) {
        for (;;) {
          int64_t ia = oa, ib = ob, id = od;
          for (int d = 0; d < nk; ++d) { ia += ki[d] * ska[d]; ib += ki[d] * skb[d]; id += ki[d] * skd[d]; }
          double ab = A[ia] * B[ib];
          double p = ab * D[id];
          s = s + p;
          int d = nk - 1;
          while (d >= 0) { if (++ki[d] < ext_k[d]) break; ki[d] = 0; --d; }
          if (d < 0) break;
        }
      }
      double as = alpha * s;
      C[oc] = (beta == 0.0) ? as : beta * C[oc] + as;
    }
    int d = nf - 1;
    while (d >= 0) { if (++fi[d] < ext_f[d]) break; fi[d] = 0; --d; }
    if (d < 0) break;
  }
}
