// tt_ws_dispatch.cu -- variant table of the warp-specialised contraction family.
#include <cuda.h>

#include "tt_launch.h"

namespace tt {

VariantInfo ws_info_w0();
VariantInfo ws_info_w1();
VariantInfo ws_info_w2();
cudaError_t ws_setup_w0();
cudaError_t ws_setup_w1();
cudaError_t ws_setup_w2();
cudaError_t ws_launch_w0(bool, bool, bool, bool, const ContractParams&, int64_t, cudaStream_t);
cudaError_t ws_launch_w1(bool, bool, bool, bool, const ContractParams&, int64_t, cudaStream_t);
cudaError_t ws_launch_w2(bool, bool, bool, bool, const ContractParams&, int64_t, cudaStream_t);

cudaError_t ws_launch_tma_w0(int, const ContractParams&, const CUtensorMap&, const CUtensorMap&, int64_t, cudaStream_t);
cudaError_t ws_launch_tma_w1(int, const ContractParams&, const CUtensorMap&, const CUtensorMap&, int64_t, cudaStream_t);
cudaError_t ws_launch_tma_w2(int, const ContractParams&, const CUtensorMap&, const CUtensorMap&, int64_t, cudaStream_t);

int num_ws_variants() { return 3; }

cudaError_t launch_contract_tma(int v, int mode, const ContractParams& p, const void* maps, int64_t nwork,
                                cudaStream_t s) {
  if (nwork <= 0) return cudaSuccess;
  const CUtensorMap* m = static_cast<const CUtensorMap*>(maps);
  return v == 0 ? ws_launch_tma_w0(mode, p, m[0], m[1], nwork, s)
       : v == 1 ? ws_launch_tma_w1(mode, p, m[0], m[1], nwork, s)
                : ws_launch_tma_w2(mode, p, m[0], m[1], nwork, s);
}

VariantInfo ws_variant_info(int v) {
  return v == 0 ? ws_info_w0() : v == 1 ? ws_info_w1() : ws_info_w2();
}

cudaError_t ws_variant_setup(int v) {
  return v == 0 ? ws_setup_w0() : v == 1 ? ws_setup_w1() : ws_setup_w2();
}

cudaError_t launch_contract_ws(int v, bool akc, bool bnc, bool av, bool bv, const ContractParams& p, int64_t nwork,
                               cudaStream_t s) {
  if (nwork <= 0) return cudaSuccess;
  return v == 0 ? ws_launch_w0(akc, bnc, av, bv, p, nwork, s)
       : v == 1 ? ws_launch_w1(akc, bnc, av, bv, p, nwork, s)
                : ws_launch_w2(akc, bnc, av, bv, p, nwork, s);
}

}  // namespace tt
