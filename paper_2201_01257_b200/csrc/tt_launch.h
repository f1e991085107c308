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
  double* P;              // split-K partial buffer (groups flagged kGroupPartial write here)
  const CGroupDesc* groups;
  const TaskDesc* tasks;
  const WorkItem* work;
  int32_t nM, nN, nK;
  double alpha, beta;
  int64_t nwork;          // work items (persistent kernels loop over them)
  int32_t sm_count;       // SMs of the device (persistent grid size)
  int32_t persistent;     // 1: grid = resident CTAs looping over items; 0: one CTA per item
  int32_t tma_n;          // TMA variant: row length of the B matrix view (N for [K][N] B, K for [N][K] B)
};

// Split-K reduction: C part = beta*C + alpha * sum_{s < nslots} P[p_off + s*vol + .] in slot order
// (deterministic, reading R12); `group` = the first chunk group (extents, strides, row range).
struct SplitDesc {
  int64_t c_off, p_off, vol;
  int32_t group, nslots;
};
cudaError_t launch_split_reduce(const double* P, double* C, const CGroupDesc* groups, const SplitDesc* splits,
                                int32_t nsplit, int32_t nM, int32_t nN, double alpha, double beta, cudaStream_t s);

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
// TMA producer variant of the warp-specialised family (uniform fused GEMM-shaped operands);
// `maps` points to two CUtensorMap (A, B).
// mode bit 0: B is [N][K] in its blocks (k contiguous); bit 1: multi-group C epilogue
cudaError_t launch_contract_tma(int v, int mode, const ContractParams& p, const void* maps, int64_t nwork,
                                cudaStream_t s);

// Segment-based element kernels (set / add / scalar / synthetic fill).
struct Segment {
  int32_t desc;       // block descriptor index
  int32_t pad;
  int64_t e0, e1;     // element range inside the block
};

// n / d for 0 <= n < 2^31 by multiply-high (Granlund-Montgomery round-up method): no integer
// division instructions in the element kernels.
struct FastDiv {
  uint32_t d, m, l;
};
inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  const uint64_t m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
  return {d, (uint32_t)m, l};
}

// Per-block descriptor for add / scalar / fill: label groups in the DESTINATION / first operand
// order (adjacent dims fused when they are adjacent and in the same order in the other operand).
struct ElemDesc {
  int64_t x_off;                        // packed offset of the block being written / walked
  int64_t y_off;                        // packed offset of the other operand's block (-1 = zero)
  int64_t g_origin;                     // global linear index of the block origin (fill)
  int32_t n;                            // number of groups
  int32_t gy;                           // transpose mode: the group with y stride 1
  int32_t mode;                         // kElemContig / kElemGeneric (segment work) or kElemTranspose
  int32_t pad;
  FastDiv div[TT_MAX_ORDER];            // group extents
  int32_t y_str[TT_MAX_ORDER];          // strides of the other operand for each group
  int64_t g_str[TT_MAX_ORDER];          // global strides (fill; groups = dims)
};

// Element-op modes: contiguous (one group, y stride 1: vectorised), generic (multiply-high decode per
// element), transpose (innermost x group strided in y: 32x32 shared-memory tiles, coalesced both
// ways), rows (innermost x group contiguous in y too: flat 16-B pairs of x, the y row base decoded per pair).
enum { kElemContig = 0, kElemGeneric = 1, kElemTranspose = 2, kElemRows = 3 };

// Transpose-mode work: one 32x32 tile of one block, bases precomputed on the host.  Element (ix, iy)
// of the tile (ix along X's contiguous group gx, iy along Y's contiguous group gy) is
// X[x_base + iy*x_ld + ix] and Y[y_base + ix*y_ld + iy].
struct TileItem {
  int64_t x_base;        // X element offset of the tile origin
  int64_t y_base;        // Y element offset of the tile origin (-1 = zero block: reads as 0)
  int32_t nx, ny;        // valid extents (<= 32) along gx / gy
  int32_t x_ld, y_ld;    // X stride of gy; Y stride of gx
};

struct ElemParams {
  double* X;
  const double* Y;
  const ElemDesc* descs;
  const Segment* segs;
  const TileItem* tiles;
  int32_t order;
  double alpha, beta;
  uint64_t key;           // fill: seed ^ tag*golden
  int32_t kind;           // fill kind
  double* partials;       // scalar: one per segment, then one per tile
};

cudaError_t launch_set(const ElemParams& p, int64_t nseg, cudaStream_t s);
// Descriptors carry their own mode: segment work (contiguous / generic descriptors) and tile work
// (transpose descriptors) of one plan run as two launches on the same stream.
cudaError_t launch_add(const ElemParams& p, int64_t nseg, int64_t ntiles, cudaStream_t s);
cudaError_t launch_fill(const ElemParams& p, int64_t nseg, cudaStream_t s);
// writes nseg + ntiles partials: p.partials[0, nseg) per segment, then one per tile
cudaError_t launch_scalar_partials(const ElemParams& p, int64_t nseg, int64_t ntiles, cudaStream_t s);
// out = alpha * sum(partials[0, n)) in a fixed order; with scratch (scalar_scratch_elems(n) doubles)
// large n is summed in two stages
int64_t scalar_scratch_elems(int64_t n);
cudaError_t launch_sum_slots(const double* part, int32_t n, double* out, cudaStream_t s);
cudaError_t launch_scalar_final(const double* partials, int64_t n, double alpha, double* out, double* scratch,
                                cudaStream_t s);

// ---- perturbative triples (NEXT-4, tt_triples.cu)
// re-tiling copy: dst block (origin, extents; dst dim order) elements <- the same global elements of src
// (another tiling and dim order: src dim q is dst dim sdim[q])
struct RetileBlk {
  int64_t dst_off;
  int32_t org[TT_MAX_ORDER];
  int32_t ext[TT_MAX_ORDER];
};
struct RetileParams {
  int32_t order;
  const double* src;
  double* dst;
  const RetileBlk* blks;
  const Segment* segs;                 // desc = RetileBlk index, [e0, e1) inside the dst block
  const int32_t* g2t[TT_MAX_ORDER];     // src tile of each global index, per src dim
  const int64_t* toff[TT_MAX_ORDER];    // src tile offsets, per src dim
  int32_t sgrid[TT_MAX_ORDER];
  int32_t sdim[TT_MAX_ORDER];
  const int64_t* sblk_off;             // src storage offsets (-1 = zero block)
};
cudaError_t launch_retile(const RetileParams& p, int64_t nseg, cudaStream_t s);

constexpr int kTripBox = 16;           // virtual box edge of the fused (T) kernel
struct TriplesParams {
  const double* VO;     // [O][O][O][V]  v^{ij}_{ma}
  const double* VV;     // [V][O][V][V]  v^{ei}_{ab}
  const double* T2;     // [O][O][V][V]  t^{ij}_{ab}
  const double* VD;     // [O][O][V][V]  v^{ij}_{ab}
  const double* T1;     // [V][O]        t^i_a
  const double* eps_o;
  const double* eps_v;
  const int2* units;    // (box triple, occupied triple)
  const int4* box3;     // box ids (a, b, c)
  const int4* trip;     // (i, j, k)
  const int32_t* box_lo;
  const int32_t* box_ext;
  int32_t nO, nV;
  int32_t o_half, v_half;   // spin split points (alpha = [0, half), R6); 0 = no spin (TMA kernel skips
                            // the spin-forbidden half of every m / e sum)
  int64_t unit0;        // first unit of this launch
  const int2* pairs;    // pair variant: (first unit, 1 or 2 units) per CTA
  double* partials;     // one per unit (indexed by unit)
  // blocked copies of the default kernel: every 8-row stage of an operand tile is ONE contiguous run
  // (1-D bulk copies), boxes of kTripBox indexed by box id, and the column index XOR-swizzled by
  // 4 (k mod 4): a half-warp's 64-bit fragment load (4 k rows x 4 columns) then touches 16 distinct
  // double banks -- conflict-free without padding
  // The summed index k runs over kp rows: each spin range [0, half) and [half, n) padded with zero rows
  // to a multiple of 8 (no spin: [0, n) padded), so every 8-row stage of a segment is one aligned run.
  // Q tiles store a stage p-major ([k/8][p][k%8][q]): a box narrower than 16 in the p role is loaded as
  // ext_p contiguous KB.
  const double* QT2;    // [z][bp][bq][m'/8][p][m'%8][q]  t^{m z}_{p q}
  const double* QVV;    // [x][bp][bq][e'/8][p][e'%8][q]  v^{e x}_{p q}
  const double* PVO;    // [x][y][br][m'][16]             v^{x y}_{m r}
  const double* PT2;    // [y][z][br][e'][16]             t^{y z}_{e r}
  int32_t nb;           // virtual boxes
  int32_t kpo, kpv;     // padded row counts m', e'
  int32_t ko2, kv2;     // first padded row of the second spin range (0 without spin)
};
// dense copy -> blocked copy (mode 0..3 = QT2, QVV, PVO, PT2)
cudaError_t launch_blockify(int mode, const TriplesParams& p, double* dst, int64_t n, cudaStream_t s);
size_t triples_fused_smem();
cudaError_t launch_triples_fused(const TriplesParams& p, int64_t nunits, cudaStream_t s);
// TMA variant; maps = 4 CUtensorMap: VO (r,m,y,x) box {20,8,1,1}, T2 as P (b,a,j,i) box {20,8,1,1},
// T2 as Q (b,a,j,i) box {18,18,1,8}, VV (q,p,x,e) box {18,18,1,8}
cudaError_t launch_triples_tma(const TriplesParams& p, int64_t nunits, cudaStream_t s);   // default kernel
// pair variant (two units with the same box triple and occupied pair (i,j) per CTA, shared operands)
cudaError_t launch_triples_pair(const TriplesParams& p, const void* maps, int64_t npairs, cudaStream_t s);
// 2-CTA cluster variant over the same pairs: the shared operand of every segment by TMA multicast
cudaError_t launch_triples_cluster(const TriplesParams& p, const void* maps, int64_t npairs, cudaStream_t s);

}  // namespace tt
