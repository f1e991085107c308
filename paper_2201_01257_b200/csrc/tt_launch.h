// tt_launch.h -- parameter blocks and launchers of the sm_100a kernels (tt_kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "tt_internal.h"

namespace tt {

constexpr int kMaxLab = 16;   // universal labels of a contraction: C labels then contracted labels

// Device task-list builder (count -> scan -> fill, canonical order R11).
struct BuildParams {
  int32_t nc, nk;                       // C dims (= C labels), contracted labels
  int32_t c_grid[TT_MAX_ORDER], k_grid[TT_MAX_ORDER];
  int32_t a_order, b_order;
  int32_t a_lab[TT_MAX_ORDER], b_lab[TT_MAX_ORDER];   // universal label of each A / B dim
  int32_t a_grid[TT_MAX_ORDER], b_grid[TT_MAX_ORDER];
  int32_t a_pos[kMaxLab], b_pos[kMaxLab];             // A / B dim of each universal label (-1 absent)
  const int64_t* lab_toff[kMaxLab];                   // tile offsets (device) of each universal label
  const uint8_t* a_nz;
  const uint8_t* b_nz;
  const int64_t* a_boff;
  const int64_t* b_boff;
  // fused groups: labels glab[first .. first+cnt) (universal indices)
  int32_t nM, nN, nK;
  int32_t m_first[kMaxGroup], m_cnt[kMaxGroup];
  int32_t n_first[kMaxGroup], n_cnt[kMaxGroup];
  int32_t k_first[kMaxGroup], k_cnt[kMaxGroup];
  int32_t glab[kMaxLab];
  const int64_t* cblocks;               // non-zero C block ids, canonical order
  int32_t ncb;
  int64_t ntuples;                      // prod k_grid
  int64_t* counts;                      // [ncb]
  int64_t* ptr;                         // [ncb + 1]
  int64_t* a_blk;                       // [ntasks]
  int64_t* b_blk;
  TaskDesc* tasks;
};

cudaError_t launch_build_count(const BuildParams& p, cudaStream_t s);
cudaError_t launch_build_scan(const BuildParams& p, cudaStream_t s);
cudaError_t launch_build_fill(const BuildParams& p, cudaStream_t s);

// Contraction kernel.
struct ContractParams {
  const double* A;
  const double* B;
  double* C;
  const CGroupDesc* groups;
  const TaskDesc* tasks;
  const WorkItem* work;
  int32_t nM, nN, nK;
  double alpha, beta;
};

struct VariantInfo {
  int bm, bn, bk, threads, smem, ctas_per_sm;
  const char* name;
};
int num_contract_variants();
VariantInfo contract_variant_info(int v);
cudaError_t launch_contract(int variant, bool a_kcontig, bool b_ncontig, const ContractParams& p,
                            int64_t nwork, cudaStream_t s);
cudaError_t contract_variant_setup(int variant);   // opt-in shared memory sizes

// Warp-specialised family (tt_contract_ws.cu): producer warps + mbarrier ring.
int num_ws_variants();
VariantInfo ws_variant_info(int v);
cudaError_t ws_variant_setup(int v);
cudaError_t launch_contract_ws(int v, bool a_kcontig, bool b_ncontig, bool a_vec, bool b_vec,
                               const ContractParams& p, int64_t nwork, cudaStream_t s);

// Segment-based element kernels (set / add / scalar / synthetic fill).
struct Segment {
  int32_t desc;       // block descriptor index
  int32_t pad;
  int64_t e0, e1;     // element range inside the block
};

// Per-block descriptor for add / scalar / fill: dims in the DESTINATION / first operand order.
struct ElemDesc {
  int64_t x_off;                        // packed offset of the block being written / walked
  int64_t y_off;                        // packed offset of the other operand's block (-1 = zero)
  int64_t g_origin;                     // global linear index of the block origin (fill)
  int32_t ext[TT_MAX_ORDER];            // block extents (x order)
  int32_t y_str[TT_MAX_ORDER];          // strides of the other operand for each x dim
  int64_t g_str[TT_MAX_ORDER];          // global strides (fill)
};

struct ElemParams {
  double* X;
  const double* Y;
  const ElemDesc* descs;
  const Segment* segs;
  int32_t order;
  double alpha, beta;
  uint64_t key;           // fill: seed ^ tag*golden
  int32_t kind;           // fill kind
  double* partials;       // scalar: one per segment
};

cudaError_t launch_set(const ElemParams& p, int64_t nseg, cudaStream_t s);
cudaError_t launch_add(const ElemParams& p, int64_t nseg, cudaStream_t s);
cudaError_t launch_fill(const ElemParams& p, int64_t nseg, cudaStream_t s);
cudaError_t launch_scalar_partials(const ElemParams& p, int64_t nseg, cudaStream_t s);
cudaError_t launch_scalar_final(const double* partials, int64_t n, double alpha, double* out,
                                cudaStream_t s);

}  // namespace tt
