// tt_host.h -- host-side helpers shared by the libtt translation units (tt_api.cpp: handles and
// layout; tt_elem.cpp: element operations; tt_contract.cpp: contraction plans, the gather and the
// partitions; tt_cholesky.cpp: the implicit Cholesky operand; tt_contract3.cpp: three-operand
// contractions; tt_triples_host.cpp: (T)).  Error reporting, workspace allocation and the plan
// cache, launch timing, label analysis, task enumeration, the gather, element and contraction plans.
// Internal: not part of the C ABI (include/tt.h).
#pragma once

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

namespace tt {

// ---------------------------------------------------------------------------------------------
// profiling scope: CUDA events around a launch on the ctx stream

struct Launch {
  tt_ctx ctx;
  std::string name;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  Launch(tt_ctx c, const char* n) : ctx(c), name(n) {
    ctx->launches++;
    ctx->last.launches++;
    if (ctx->profiling) {
      e0 = get_event();
      e1 = get_event();
      cudaEventRecord(e0, ctx->stream);
    }
  }
  cudaEvent_t get_event() {
    if (!ctx->event_pool.empty()) {
      cudaEvent_t e = ctx->event_pool.back();
      ctx->event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  ~Launch() {
    if (ctx->profiling) {
      cudaEventRecord(e1, ctx->stream);
      ctx->prof.push_back({name, e0, e1});
    }
  }
};

tt_status nccl_check(int r, const char* what);
// ---------------------------------------------------------------------------------------------
// label analysis (P145-174; S356-384, S412-413)

struct Analysis {
  std::string c, a, b;
  int nc = 0, nk = 0;
  std::vector<char> uni;                 // universal labels: C labels, then contracted (A order)
  std::vector<int> a_lab, b_lab;         // universal label of each A / B dim
  std::vector<int> a_pos, b_pos, c_pos;  // dim of each universal label in A / B / C (-1)
  std::vector<std::vector<int>> mg, ng, kg;
  bool a_kc = true, b_nc = true;
};

bool same_tiling(tt_tis x, tt_tis y);
tt_status check_labels(const char* lbl, tt_tensor t, const char* which);
tt_status tiling_of(const Analysis& an, char x, tt_tensor C, tt_tensor A, tt_tensor B, tt_tis* out);
tt_status analyse(tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B, const char* bl,
                  Analysis& an);
int n_variants();
VariantInfo variant_info(int v);
double variant_efficiency(int v, bool tma);
tt_tis label_tis(const Analysis& an, int u, tt_tensor C, tt_tensor A);
// ---------------------------------------------------------------------------------------------
// host canonical task list (reading R11)

struct HostTasks {
  std::vector<int64_t> cblk, ptr, a_blk, b_blk, cost;
  std::vector<int32_t> K;     // contracted extent per task
};

void enumerate_tasks(const Analysis& an, tt_tensor C, tt_tensor A, tt_tensor B, HostTasks& ht);
std::vector<int32_t> lpt(const std::vector<int64_t>& cost, const std::vector<int64_t>& ids, int nranks);
// ---------------------------------------------------------------------------------------------
// gather plan: element ranges of input blocks this rank reads but does not hold (P212; SURVEY
// §8(a) A4).  A need is a range [e0, e1) of a block (the whole block, or the rows of a row-split
// part); the sources are the block's owner or the owners of the overlapping parts.

struct Run {
  int op;        // operand index into the ops list
  int peer;
  int64_t off, len;
};

struct GatherPlan {
  std::vector<int64_t> recv_list, send_list;   // (op, block, peer, e0, e1) rows
  std::vector<Run> recv, send;
  int64_t recv_bytes = 0;
  int64_t all_pieces = 0;   // pieces over ALL ranks: 0 = no rank exchanges anything (same on every rank)
  bool one_group = false;   // few pieces over ALL ranks (the same decision on every rank): one NCCL group
};

struct Need {
  int op;
  int64_t blk, e0, e1;
};

using Needs = std::vector<std::vector<Need>>;   // per rank

void normalize(std::vector<Need>& v);
// owners of the pieces of [e0, e1) of block b of T
template <class F>
void pieces(tt_tensor T, int64_t b, int64_t e0, int64_t e1, F&& emit) {
  if (T->parts[b].empty()) {
    emit(T->owner[b], e0, e1);
    return;
  }
  const int64_t inner = T->block_volume(b) / T->ext0(b);
  for (const auto& p : T->parts[b]) {
    const int64_t a = std::max(e0, p.lo * inner), z = std::min(e1, p.hi * inner);
    if (a < z) emit(p.owner, a, z);
  }
}

constexpr size_t kGatherGroupOps = 128;   // NCCL point-to-point calls per group and direction

tt_status build_gather(tt_ctx ctx, Needs need, const std::vector<tt_tensor>& ops, GatherPlan& gp);
tt_status wait_comm(tt_ctx ctx);
tt_status sim_exchange(tt_ctx ctx, const GatherPlan& gp, const std::vector<tt_tensor>& ops, cudaStream_t stream);
tt_status allreduce_sum(tt_ctx ctx, double* dst, cudaStream_t stream);
tt_status run_gather(tt_ctx ctx, const GatherPlan& gp, const std::vector<tt_tensor>& ops,
                     cudaStream_t stream = nullptr);
tt_status ensure_dev(tt_tensor t);
tt_status check_bound(tt_tensor t, const char* which);
// ---------------------------------------------------------------------------------------------
// contraction plan (cached per (tensors, owner versions, labels))

// Internal contraction options (used by the implicit-operand driver): `local` plans compute exactly
// the listed C parts of this rank and never gather (the operands are local / replicated);
// `no_gather` plans list this rank's C parts (ownership) but build no gather (accounting plans of
// the implicit-operand driver, which moves its operands itself).
struct PartSel {
  int64_t blk, lo, hi;
};

struct ContractOpts {
  bool local = false;
  bool no_gather = false;
  std::vector<PartSel> sel;
  std::string tag;
  int force_variant = -1;   // autotuning: build this kernel variant instead of the model's choice
};

struct ContractPlan {
  DevMem mem;                          // workspace regions of the device arrays below
  Analysis an;
  HostTasks ht;
  struct MyPart {
    int g;                         // index into ht.cblk
    int64_t lo, hi;                // rows of the block's dim-0 tile computed by this rank
  };
  std::vector<MyPart> my;
  GatherPlan gp;
  int variant = 0;
  bool a_vec = false, b_vec = false;   // 16-byte copies along the operand's contiguous direction
  bool persistent = false;             // short work items: persistent CTAs hide pipeline fill / epilogue
  bool tma = false;                    // TMA producer (uniform fused GEMM-shaped operands)
  int64_t tma_k = 0, tma_n = 0;        // row lengths of the A [rows][K] and B [rows][N|K] views
  int tma_mode = 0;                    // bit 0: B is [N][K]; bit 1: multi-group C epilogue
  CUtensorMap maps[2];                 // A, B tensor maps (encoded for map_ptr)
  const void* map_ptr[2] = {nullptr, nullptr};
  int64_t nwork = 0;
  CGroupDesc* d_groups = nullptr;
  TaskDesc* d_tasks = nullptr;
  WorkItem* d_work = nullptr;
  std::vector<SplitDesc> splits;       // split-K parts (reduced after the GEMM kernel)
  SplitDesc* d_splits = nullptr;
  double* d_partials = nullptr;        // their partial sums, one slot per chunk
  int64_t partial_elems = 0;
  int64_t* d_ablk = nullptr;
  int64_t* d_bblk = nullptr;
  int64_t* d_ptr = nullptr;
  bool device_built = false;
  int alt_variant = -1;                // runner-up of the variant model (warp-specialised family)
  int tune = 0;                        // autotuning state: 0 untimed, 1 main timed, 2 decided
  float tune_ms = 0;
  std::shared_ptr<ContractPlan> alt;   // the same plan built for alt_variant
  bool use_alt = false;
  cudaEvent_t pf_event = nullptr;      // tt_contract_prefetch: this plan's gather issued on the comm stream
  bool prefetched = false;
  double flops = 0, bytes = 0;
  int64_t tasks = 0;
  // wave tail: the last work items (less than one wave of resident CTAs) re-tiled with the smallest
  // warp-specialised tile and launched right after the main kernel, one small CTA per idle SM
  int tail_variant = -1;
  int64_t tail_nwork = 0;
  CGroupDesc* d_tail_groups = nullptr;
  WorkItem* d_tail_work = nullptr;
  CUtensorMap tail_maps[2];
  const void* tail_map_ptr[2] = {nullptr, nullptr};
};

std::string plan_key(const char* kind, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                     const char* bl, double beta);
#define TT_CUDA(x)                                                                    \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) return fail(TT_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

#define TT_TRY(x)                 \
  do {                            \
    tt_status s_ = (x);           \
    if (s_ != TT_OK) return s_;   \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  bool active = false;
  explicit DeviceGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      cudaSetDevice(dev);
      active = true;
    }
  }
  ~DeviceGuard() {
    if (active) cudaSetDevice(prev);
  }
};

tt_status need_device(tt_ctx ctx);
tt_status need_ws(tt_ctx ctx);
template <class T>
tt_status dev_alloc(tt_ctx ctx, DevMem& m, T** p, size_t n) {
  void* v = nullptr;
  *p = nullptr;
  TT_TRY(ws_alloc(ctx, m, (int64_t)(std::max<size_t>(n, 1) * sizeof(T)), &v));
  *p = (T*)v;
  return TT_OK;
}

void plan_put(tt_ctx ctx, const std::string& key, std::shared_ptr<void> p);
bool evict_one(tt_ctx ctx);
tt_status drain_retired(tt_ctx ctx);
tt_status ws_make_room(tt_ctx ctx);
extern thread_local std::string g_err;
extern std::atomic<uint64_t> g_uid;
tt_status fail(tt_status code, const char* fmt, ...);
constexpr int64_t kSegElems = 1 << 15;

struct ElemPlan {
  DevMem mem;                 // workspace regions of the device arrays below
  std::vector<ElemDesc> descs;
  std::vector<Segment> segs;
  std::vector<TileItem> tiles;
  ElemDesc* d_descs = nullptr;
  Segment* d_segs = nullptr;
  TileItem* d_tiles = nullptr;
  double* d_partials = nullptr;
  GatherPlan gp;
  double bytes = 0;
  int64_t blocks = 0;
  int64_t nseg() const { return (int64_t)segs.size(); }
  int64_t ntiles() const { return (int64_t)tiles.size(); }
};

int fuse_elem(ElemDesc& d, int order, const int32_t* ext, const int* ypos, const int64_t* ystr);
void add_tiles(ElemPlan& ep, const ElemDesc& d);
void add_segments(ElemPlan& ep, int32_t desc, int64_t e_begin, int64_t e_end);
void emit_elem(ElemPlan& ep, ElemDesc& d, bool whole, const std::vector<std::pair<int64_t, int64_t>>& ranges);
int64_t sub_range_inner(tt_tensor Y, int64_t yb, bool same_dim0, int64_t lo_row, int64_t hi_row, int64_t* e0,
                        int64_t* e1);
tt_status upload_elem_once(tt_ctx ctx, ElemPlan& ep, bool partials);
tt_status upload_elem(tt_ctx ctx, ElemPlan& ep, bool partials);
template <class P>
std::shared_ptr<P> cached(tt_ctx ctx, const std::string& key) {
  auto it = ctx->plans.find(key);
  if (it == ctx->plans.end()) return nullptr;
  it->second.tick = ++ctx->plan_tick;
  if (ctx->plan_sink) ctx->plan_sink->push_back(it->second.p);
  return std::static_pointer_cast<P>(it->second.p);
}

void reset_stats(tt_ctx ctx);
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn();
tt_status encode_2d(CUtensorMap* m, const double* base, int64_t cols, int64_t rows, uint32_t box_cols, uint32_t box_rows,
                    bool swizzle128);
tt_status encode_3d(CUtensorMap* m, const double* base, const int64_t* dims3, const uint32_t* box3);
tt_status encode_4d(CUtensorMap* m, const double* base, const int64_t* dims4, const uint32_t* box4);
int64_t uniform_group_extent(tt_tensor T, const std::vector<int>& tdims);
tt_status build_contract_plan(tt_ctx ctx, tt_tensor C, tt_tensor A, tt_tensor B, double beta, ContractPlan& pl,
                              const ContractOpts& opts = ContractOpts());
tt_status get_contract_plan(tt_ctx ctx, tt_tensor C, const char* cl, tt_tensor A, const char* al, tt_tensor B,
                            const char* bl, double beta, std::shared_ptr<ContractPlan>& out, bool* cached_flag,
                            const ContractOpts& opts = ContractOpts());
tt_status launch_plan(tt_ctx ctx, const ContractPlan& pl, tt_tensor C, const char* cl, double beta, double alpha,
                      tt_tensor A, const char* al, tt_tensor B, const char* bl);

// tensor layout helpers (tt_api.cpp): a parent's layout is frozen while views live; storage offsets
// (global or compact); the row-part view of a tensor's parts
tt_status check_no_views(tt_tensor t);
void apply_storage(tt_tensor t);
void refresh_parts_view(tt_tensor t);
// a tensor handle with dims and block count set (tensor_new), then its layout from the block map
// (tensor_finish)
tt_status tensor_new(tt_ctx ctx, int32_t order, const tt_tis* dims, tt_tensor* out);
void tensor_finish(tt_tensor t);

// implicit Cholesky operand (tt_cholesky.cpp): the block maps of V and W from X's, the argument
// checks, and a metadata-only tensor (no storage) over given dims and block map
void chol_maps(tt_tensor X, const std::vector<tt_tis>& vd, std::vector<uint8_t>& vnz, std::vector<uint8_t>& wnz);
tt_status chol_check(tt_tensor C, const char* cl, tt_tensor X, const char* vl, tt_tensor B, const char* bl,
                     std::vector<tt_tis>& vd);
tt_status new_meta_tensor(tt_ctx ctx, const std::vector<tt_tis>& dims, const std::vector<uint8_t>& nz, tt_tensor* out);

}  // namespace tt
