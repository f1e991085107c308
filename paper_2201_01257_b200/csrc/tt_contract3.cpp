// tt_contract3.cpp -- three-operand contraction through an intermediate (PAPER Eqs. cc9-cc11, P293-311).  Citations as in include/tt.h.
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
// three-operand contraction evaluated through an intermediate (PAPER Eqs.
// cc9-cc11, P293-311: the n_o^4 n_u^4 term 1/4 v^{ef}_{mn} t^{ij}_{ef} t^{mn}_{ab} becomes
// I^{ij}_{mn} = v^{ef}_{mn} t^{ij}_{ef} followed by 1/4 I^{ij}_{mn} t^{mn}_{ab}, "total numerical cost
// proportional to n_o^4 n_u^2").  Every pairing is costed on the block maps (reading R26) and the
// cheapest is executed as two binary contractions of the DMMA path.

namespace {

struct C3Plan {
  tt_tensor I = nullptr;
  std::string i_lbl, x_lbl, y_lbl, z_lbl;
  int pair = 0;
  tt_tensor X = nullptr, Y = nullptr, Z = nullptr;
  double flops[3] = {0, 0, 0}, naive = 0;
  ~C3Plan() { delete I; }
};

struct C3Cand {
  std::string il;
  std::vector<tt_tis> idims;
  std::vector<uint8_t> inz;
  double flops1 = 0, flops2 = 0;
};

// intermediate of the pair (X, Y) when the third operand is Z: the labels of X then Y that survive
// (appear in Z or in C), on their tiled spaces; its block map = the blocks that receive a task.
tt_status c3_candidate(tt_ctx ctx, tt_tensor C, const std::string& cl, tt_tensor X, const std::string& xl,
                       tt_tensor Y, const std::string& yl, tt_tensor Z, const std::string& zl, C3Cand& cd) {
  cd.il.clear();
  cd.idims.clear();
  for (int s = 0; s < 2; ++s) {
    const std::string& l = s ? yl : xl;
    tt_tensor T = s ? Y : X;
    for (size_t d = 0; d < l.size(); ++d) {
      const char x = l[d];
      const bool keep = zl.find(x) != std::string::npos || cl.find(x) != std::string::npos;
      if (keep && cd.il.find(x) == std::string::npos) {
        cd.il.push_back(x);
        cd.idims.push_back(T->dims[d]);
      }
    }
  }
  if (cd.il.empty() || cd.il.size() > (size_t)TT_MAX_ORDER)
    return fail(TT_E_UNSUPPORTED, "intermediate of order %zu", cd.il.size());
  tt_tensor Id;
  int64_t nb = 1;
  for (auto d : cd.idims) nb *= d->ntiles();
  TT_TRY(new_meta_tensor(ctx, cd.idims, std::vector<uint8_t>(nb, 1), &Id));
  std::unique_ptr<tt_tensor_s> hold(Id);
  Analysis a1;
  TT_TRY(analyse(Id, cd.il.c_str(), X, xl.c_str(), Y, yl.c_str(), a1));
  HostTasks h1;
  enumerate_tasks(a1, Id, X, Y, h1);
  cd.inz.assign(nb, 0);
  cd.flops1 = 0;
  for (size_t g = 0; g < h1.cblk.size(); ++g)
    if (h1.ptr[g + 1] > h1.ptr[g]) {
      cd.inz[h1.cblk[g]] = 1;
      cd.flops1 += (double)h1.cost[g];
    }
  Id->nz = cd.inz;
  tensor_finish(Id);
  Analysis a2;
  TT_TRY(analyse(C, cl.c_str(), Id, cd.il.c_str(), Z, zl.c_str(), a2));
  HostTasks h2;
  enumerate_tasks(a2, C, Id, Z, h2);
  cd.flops2 = 0;
  for (int64_t c : h2.cost) cd.flops2 += (double)c;
  return TT_OK;
}

// multiply-adds of the unfactorized loop: one product A*B*D per combination of all label values whose
// four blocks (C, A, B, D) are non-zero; -1 when the label tile grid is too large to enumerate
double c3_naive_macs(tt_tensor C, const std::string& cl, tt_tensor const T[3], const std::string L[3]) {
  std::string uni = cl;
  std::vector<tt_tis> lt;
  for (size_t d = 0; d < cl.size(); ++d) lt.push_back(C->dims[d]);
  for (int s = 0; s < 3; ++s)
    for (size_t d = 0; d < L[s].size(); ++d)
      if (uni.find(L[s][d]) == std::string::npos) { uni.push_back(L[s][d]); lt.push_back(T[s]->dims[d]); }
  double ntup = 1;
  for (auto t : lt) ntup *= t->ntiles();
  if (ntup > 5e7) return -1;
  const int nu = (int)uni.size();
  std::vector<int32_t> tile(nu, 0);
  double macs = 0;
  for (int64_t k = 0; k < (int64_t)ntup; ++k) {
    int64_t r = k;
    for (int u = nu - 1; u >= 0; --u) { tile[u] = (int32_t)(r % lt[u]->ntiles()); r /= lt[u]->ntiles(); }
    auto nzof = [&](tt_tensor T, const std::string& l) {
      int64_t b = 0;
      for (size_t d = 0; d < l.size(); ++d) b = b * T->grid[d] + tile[uni.find(l[d])];
      return T->nz[b] != 0;
    };
    if (!nzof(C, cl) || !nzof(T[0], L[0]) || !nzof(T[1], L[1]) || !nzof(T[2], L[2])) continue;
    double v = 1;
    for (int u = 0; u < nu; ++u) v *= (double)lt[u]->size(tile[u]);
    macs += v;
  }
  return macs;
}

}  // namespace

extern "C" {

tt_status tt_contract3(tt_ctx ctx, tt_tensor C, const char* cl, double beta, double alpha, tt_tensor A,
                       const char* al, tt_tensor B, const char* bl, tt_tensor D, const char* dl, void* workspace,
                       int64_t ws_elems, tt_contract3_info* info) {
  NvtxRange nvtx_("tt_contract3");
  if (!ctx || !C || !A || !B || !D || !cl || !al || !bl || !dl) return fail(TT_E_ARG, "NULL argument");
  TT_TRY(check_labels(cl, C, "C"));
  TT_TRY(check_labels(al, A, "A"));
  TT_TRY(check_labels(bl, B, "B"));
  TT_TRY(check_labels(dl, D, "D"));
  const std::string L[4] = {cl, al, bl, dl};
  // every label in exactly two of the four operands (no batch / dangling labels, S380)
  for (int s = 0; s < 4; ++s)
    for (char x : L[s]) {
      int n = 0;
      for (int q = 0; q < 4; ++q) n += L[q].find(x) != std::string::npos;
      if (n != 2) return fail(TT_E_LABEL, "label '%c' appears in %d of C, A, B, D (must be exactly 2)", x, n);
    }
  char keybuf[600];
  snprintf(keybuf, sizeof(keybuf), "c3|%llu.%llu|%llu.%llu|%llu.%llu|%llu.%llu|%s|%s|%s|%s",
           (unsigned long long)C->uid, (unsigned long long)C->version, (unsigned long long)A->uid,
           (unsigned long long)A->version, (unsigned long long)B->uid, (unsigned long long)B->version,
           (unsigned long long)D->uid, (unsigned long long)D->version, cl, al, bl, dl);
  auto cp = cached<C3Plan>(ctx, keybuf);
  double cand_flops[3] = {0, 0, 0};
  double naive = 0;
  if (!cp) {
    cp = std::make_shared<C3Plan>();
    tt_tensor T[3] = {A, B, D};
    const std::string TL[3] = {al, bl, dl};
    static const int pairs[3][3] = {{0, 1, 2}, {0, 2, 1}, {1, 2, 0}};   // (X, Y, Z): (AB)D, (AD)B, (BD)A
    C3Cand best;
    int bi = -1;
    for (int p = 0; p < 3; ++p) {
      const int x = pairs[p][0], y = pairs[p][1], z = pairs[p][2];
      C3Cand cd;
      tt_status st = c3_candidate(ctx, C, cl, T[x], TL[x], T[y], TL[y], T[z], TL[z], cd);
      if (st == TT_E_UNSUPPORTED) { cand_flops[p] = -1; continue; }
      TT_TRY(st);
      cand_flops[p] = cd.flops1 + cd.flops2;
      if (bi < 0 || cand_flops[p] < cand_flops[bi]) { bi = p; best = cd; }
    }
    if (bi < 0) return fail(TT_E_UNSUPPORTED, "no pairing has a supported intermediate");
    naive = c3_naive_macs(C, cl, T, TL);
    cp->pair = bi;
    cp->X = T[pairs[bi][0]]; cp->x_lbl = TL[pairs[bi][0]];
    cp->Y = T[pairs[bi][1]]; cp->y_lbl = TL[pairs[bi][1]];
    cp->Z = T[pairs[bi][2]]; cp->z_lbl = TL[pairs[bi][2]];
    cp->i_lbl = best.il;
    TT_TRY(new_meta_tensor(ctx, best.idims, best.inz, &cp->I));
    cp->I->ctx = ctx;
    // remember the costs with the plan (returned on every call)
    cp->flops[0] = cand_flops[0]; cp->flops[1] = cand_flops[1]; cp->flops[2] = cand_flops[2];
    cp->naive = naive;
    plan_put(ctx, keybuf, cp);
  }
  const int64_t need = (cp->I->storage_elems + 1) / 2 * 2;
  if (info) {
    info->pair = cp->pair;
    memset(info->i_lbl, 0, sizeof(info->i_lbl));
    memcpy(info->i_lbl, cp->i_lbl.data(), cp->i_lbl.size());
    for (int p = 0; p < 3; ++p) info->flops[p] = cp->flops[p];
    info->naive_macs = cp->naive;
    info->ws_elems = need;
  }
  if (!workspace) return TT_OK;   // query: pairing, costs and workspace size only
  if (ws_elems < need) return fail(TT_E_ARG, "workspace holds %lld doubles, the intermediate needs %lld",
                                   (long long)ws_elems, (long long)need);
  TT_TRY(tt_tensor_bind(cp->I, workspace, ws_elems));
  TT_TRY(tt_contract(ctx, cp->I, cp->i_lbl.c_str(), 0.0, 1.0, cp->X, cp->x_lbl.c_str(), cp->Y, cp->y_lbl.c_str()));
  const tt_stats first = ctx->last;
  TT_TRY(tt_contract(ctx, C, cl, beta, alpha, cp->I, cp->i_lbl.c_str(), cp->Z, cp->z_lbl.c_str()));
  ctx->last.flops += first.flops;
  ctx->last.tasks += first.tasks;
  ctx->last.gathered_bytes += first.gathered_bytes;
  ctx->last.bytes += first.bytes;
  return TT_OK;
}

}  // extern "C"
