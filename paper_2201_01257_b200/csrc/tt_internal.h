// tt_internal.h -- internal types of libtt (host metadata + device descriptors).
// Not part of the ABI (include/tt.h is).  Citations as in tt.h.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <map>
#include <set>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/tt.h"

namespace tt {

constexpr int kMaxGroup = 4;  // fused label groups per GEMM side (M, N, K)

// ------------------------------------------------------------------------------------------------
// Device descriptors (built on device by the task builder, read by the contraction kernel).

// One per non-zero C block this rank computes.  GEMM view of the block:
// m = mixed radix over the fused M groups (labels of C that come from A, C order), n over the
// fused N groups (labels from B), innermost last.
constexpr int32_t kGroupPartial = 1;

struct CGroupDesc {
  int64_t c_off;                 // packed offset of the C block
  int32_t M, N;                  // GEMM row / column END of this group (exclusive)
  int32_t m_begin, n_begin;      // first row / column (a part of a row-split block; else 0)
  int32_t task_begin, task_end;  // CSR range in the task array
  int32_t nstages;               // sum over tasks of ceil(K_t / BK) for the chosen kernel BK
  int32_t flags;                 // kGroupPartial: a split-K chunk writing raw sums into the partial
                                 // buffer (c_off is then an offset into ContractParams::P)
  int32_t mext[kMaxGroup], next[kMaxGroup];     // fused group extents
  int32_t cm_str[kMaxGroup], cn_str[kMaxGroup]; // their strides inside the C block
};

// One per non-zero (A block, B block) pair.
struct TaskDesc {
  int64_t a_off, b_off;          // packed offsets of the A and B blocks
  int32_t K;                     // contracted extent of this pair
  int32_t pad;
  int32_t kext[kMaxGroup];                      // fused K group extents (order of first appearance in A)
  int32_t ak_str[kMaxGroup], bk_str[kMaxGroup]; // K group strides in the A / B block
  int32_t am_str[kMaxGroup], bn_str[kMaxGroup]; // M group strides in A, N group strides in B
};

// sets the thread-local error message of tt_last_error and returns `code`
tt_status set_error(tt_status code, const char* msg);

struct WorkItem {
  int32_t group;   // index into CGroupDesc array
  int32_t mt, nt;  // tile coordinates inside the block
};

// Label analysis of a contraction after fusing adjacent labels (DESIGN.md §5 "label fusion").
struct LabelGroup {
  std::vector<int> labels;  // original label chars (as ints), in group order
};

struct ContractionShape {
  std::string c_lbl, a_lbl, b_lbl;
  std::vector<char> con;                   // contracted labels, order of first appearance in A
  std::vector<LabelGroup> mg, ng, kg;      // fused groups
  bool a_kcontig = true;                   // A's innermost label is a K label
  bool b_ncontig = true;                   // B's innermost label is an N label
};

// ------------------------------------------------------------------------------------------------
// Device workspace (tt_workspace_bind; SURVEY §8(b), P182-186 "ExecutionContext ... memory manager"):
// ONE caller-owned device buffer per context from which all library metadata (tensor block maps, task
// descriptors, work lists, element-op segments) and scratch (split-K partials, scalar partials) are
// carved.  There is no cudaMalloc on the execute path.  Host-side first-fit allocator over offsets with
// coalescing; released regions are "retired" until the device has drained (they may still be read by
// queued kernels) and become reusable after one device synchronisation.  When the buffer is full the
// context evicts least-recently-used cached plans that nobody else references.
constexpr int64_t kWsAlign = 256;
constexpr int64_t kWsMin = 1 << 20;   // tt_workspace_bytes before any call

struct Arena {
  char* base = nullptr;
  int64_t size = 0;
  std::map<int64_t, int64_t> free_;                     // offset -> length, coalesced
  std::vector<std::pair<int64_t, int64_t>> retired;     // released, reusable after a device drain
  int64_t live = 0, high = 0, need = 0;                 // bytes in use, high-water, failed-call need
  uint64_t gen = 0;                                     // bumped at every bind
  void reset(char* b, int64_t n) {
    base = b;
    size = n;
    free_.clear();
    retired.clear();
    if (n > 0) free_[0] = n;
    live = high = need = 0;
    ++gen;
  }
  // first fit from the bottom (plans: short-lived, evictable), or last fit from the top (long-lived
  // tensor metadata and scratch), so that the pinned regions do not fragment the plans' space
  bool take(int64_t n, int64_t* off, bool top = false) {
    auto fits = [&](std::map<int64_t, int64_t>::iterator it) {
      const int64_t blo = it->first, blen = it->second;
      *off = top ? blo + blen - n : blo;
      free_.erase(it);
      if (top) {
        if (blen > n) free_[blo] = blen - n;
      } else if (blen > n) {
        free_[blo + n] = blen - n;
      }
      live += n;
      if (live > high) high = live;
      return true;
    };
    if (top) {
      for (auto it = free_.end(); it != free_.begin();) {
        --it;
        if (it->second >= n) return fits(it);
      }
      return false;
    }
    for (auto it = free_.begin(); it != free_.end(); ++it)
      if (it->second >= n) return fits(it);
    return false;
  }
  void give(int64_t off, int64_t n) {                   // back to the free list, coalescing
    auto it = free_.emplace(off, n).first;
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_.erase(nx);
    }
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_.erase(it);
      }
    }
  }
};

// The regions one owner (a plan, a tensor's device metadata, the context scratch) holds in the
// workspace; retired when the owner is destroyed.
struct DevMem {
  tt_ctx ctx = nullptr;
  uint64_t gen = 0;
  bool top = false;            // long-lived owner: allocated from the top of the workspace
  std::vector<std::pair<int64_t, int64_t>> regions;
  DevMem() = default;
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  explicit DevMem(bool long_lived) : top(long_lived) {}
  DevMem(DevMem&& o) noexcept : ctx(o.ctx), gen(o.gen), top(o.top), regions(std::move(o.regions)) { o.regions.clear(); }
  DevMem& operator=(DevMem&& o) noexcept {
    if (this != &o) {
      release();
      ctx = o.ctx;
      gen = o.gen;
      top = o.top;
      regions = std::move(o.regions);
      o.regions.clear();
    }
    return *this;
  }
  ~DevMem() { release(); }
  void release();              // retire every region (tt_api.cpp)
  void forget() { regions.clear(); }   // the arena is being reset: nothing to give back
};

tt_status ws_alloc(tt_ctx ctx, DevMem& m, int64_t bytes, void** out);

}  // namespace tt

// ------------------------------------------------------------------------------------------------
// Host handle types.

struct tt_is_s {
  int64_t extent = 0;
  std::vector<int64_t> rb, re;   // ranges [rb, re)
  std::vector<int8_t> rspin;
};

struct tt_tis_s {
  tt_is is = nullptr;
  std::vector<int64_t> offsets;  // ntiles + 1
  std::vector<int8_t> spin;      // per tile
  uint64_t uid = 0;
  tt_tis parent = nullptr;       // sub-space (tt_tis_sub / tt_tis_range): the tiled space it slices
  int32_t tile0 = 0;             // ... and the parent tile index of its tile 0
  int32_t ntiles() const { return (int32_t)offsets.size() - 1; }
  int64_t size(int t) const { return offsets[t + 1] - offsets[t]; }
};

struct tt_tensor_s {
  tt_ctx ctx = nullptr;
  uint64_t seq = 0;                // creation index in its context (SPMD: same tensor, same seq on every rank)
  tt_sim sim = nullptr;            // simulated-rank group of its context (registry entry), else nullptr
  int32_t sim_rank = 0;
  int32_t order = 0;
  std::vector<tt_tis> dims;
  std::vector<int32_t> grid;       // ntiles per dim
  int64_t nblocks = 0, nnz = 0;
  std::vector<uint8_t> nz;
  std::vector<int64_t> blk_off;    // STORAGE offsets (= gblk_off unless compact; -1 = not stored)
  std::vector<int64_t> gblk_off;   // global packed offsets (R10)
  std::vector<int32_t> owner;
  int64_t packed_elems = 0;
  bool compact = false;            // storage holds only this rank's held ranges (tt_tensor_set_compact)
  int64_t storage_elems = 0;       // doubles the bound buffer must hold
  double* data = nullptr;
  int64_t capacity = 0;
  uint64_t uid = 0;
  uint64_t version = 0;            // bumped when the owner map changes (plan cache key)
  // device metadata (lazily uploaded)
  uint8_t* d_nz = nullptr;
  int64_t* d_blk_off = nullptr;
  std::vector<int64_t*> d_toff;   // per dim tile offsets on the device
  tt::DevMem mem{true};            // workspace regions of the device metadata above (long-lived)
  bool dev_ready = false;
  bool dev_off_stale = false;      // storage offsets changed since the last upload
  // row-range ownership (SURVEY §8(e) block splitting): a split block is owned by parts, each a
  // range [lo, hi) of the block's dimension-0 tile; owner[b] is then TT_SPLIT
  struct Part {
    int32_t lo, hi, owner;
  };
  std::vector<std::vector<Part>> parts;     // per block; empty = whole block owned by owner[b]
  std::vector<int64_t> pv_blk;              // flattened view for tt_tensor_parts
  std::vector<int32_t> pv_lo, pv_hi, pv_owner;
  bool any_split = false;
  tt_tensor view_of = nullptr;     // sliced view (tt_tensor_view): blocks live in this tensor's storage
  int32_t live_views = 0;          // views of this tensor not yet destroyed: its layout is frozen meanwhile

  ~tt_tensor_s();                  // leaves the context's tensor registry (tt_api.cpp)
  int64_t ext0(int64_t b) const {
    int32_t c[TT_MAX_ORDER];
    block_coords(b, c);
    return dims[0]->size(c[0]);
  }
  // element ranges [e0, e1) of block b held by `rank` (whole block, replicated, or its parts)
  void held_ranges(int64_t b, int32_t rank, std::vector<std::pair<int64_t, int64_t>>& out) const {
    out.clear();
    if (!nz[b]) return;
    if (parts[b].empty()) {
      if (owner[b] == rank || owner[b] == TT_REPLICATED) out.push_back({0, block_volume(b)});
      return;
    }
    const int64_t inner = block_volume(b) / ext0(b);
    for (const Part& p : parts[b])
      if (p.owner == rank) out.push_back({p.lo * inner, p.hi * inner});
  }
  bool held(int64_t b, int32_t rank) const { return nz[b] && (owner[b] == rank || owner[b] == TT_REPLICATED); }

  void block_coords(int64_t b, int32_t* c) const {
    for (int d = order - 1; d >= 0; --d) { c[d] = (int32_t)(b % grid[d]); b /= grid[d]; }
  }
  int64_t block_id(const int32_t* c) const {
    int64_t b = 0;
    for (int d = 0; d < order; ++d) b = b * grid[d] + c[d];
    return b;
  }
  int64_t block_volume(int64_t b) const {
    int32_t c[TT_MAX_ORDER];
    block_coords(b, c);
    int64_t v = 1;
    for (int d = 0; d < order; ++d) v *= dims[d]->size(c[d]);
    return v;
  }
};

// NVTX range per ABI call (visible in nsys / ncu --nvtx-include); header-only NVTX v3 (dlopen-based)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct ProfileRec {
  std::string name;
  cudaEvent_t e0, e1;
};

struct tt_ctx_s {
  int32_t device = -1;
  cudaStream_t stream = nullptr;
  int32_t rank = 0, nranks = 1;
  void* comm = nullptr;            // ncclComm_t
  bool profiling = false;
  std::vector<ProfileRec> prof;
  std::vector<cudaEvent_t> event_pool;
  int64_t launches = 0;
  tt_stats last{};
  struct PlanEntry {
    std::shared_ptr<void> p;
    uint64_t tick = 0;                                   // last use (LRU eviction)
  };
  std::map<std::string, PlanEntry> plans;                // plan cache (type-erased)
  uint64_t plan_tick = 0;
  int64_t plan_limit = 1 << 14;                          // cached plans kept at most (tt_ctx_set_plan_limit)
  std::vector<std::shared_ptr<void>>* plan_sink = nullptr;   // scheduler capture: keeps every plan it uses alive
  int32_t graph_pins = 0;                                // captured graphs reading workspace pointers
  tt::Arena ws;                                          // the bound device workspace
  tt::DevMem scratch{true};                              // context scratch (d_scalar)
  std::set<tt_tensor_s*> tensors;                        // live tensors (their metadata lives in ws)
  double* d_scalar = nullptr;                            // scratch for scalar results
  double* d_partials = nullptr;
  int32_t sm_count = 148;
  // scheduler support: build plans without launching (graph capture preparation), and write scalar
  // results to a device slot instead of the host (inside a captured graph)
  bool prepare_only = false;
  double* scalar_dev_out = nullptr;
  // prefetched input gathers (tt_contract_prefetch): NCCL on a side stream, overlapping earlier kernels
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t comm_fork = nullptr, comm_done = nullptr;
  bool comm_pending = false;       // comm_done marks the last gather issued on comm_stream
  // tt_contract_host: host<->device copies overlapping the contraction tiles
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_fork = nullptr;
  std::vector<cudaEvent_t> tile_events;
  // simulated ranks on one GPU (tt_ctx_create_sim): the group replacing the NCCL communicator
  tt_sim sim = nullptr;
  uint64_t tensor_seq = 0;         // next tensor creation index
};

// Simulated ranks: nranks contexts on ONE device, each driven by its
// own host thread exactly as one process per GPU would be (SPMD).  Collectives: a host barrier over
// the group plus CUDA events: the gather becomes one cudaMemcpyAsync (device to device) per run from
// the peer's buffer, the all-reduce a fixed-rank-order sum of the ranks' partials.
struct tt_sim_s {
  int32_t nranks = 0, device = -1;
  std::vector<tt_ctx> ctx;                        // registered contexts by rank
  std::vector<cudaEvent_t> ready, done;           // per rank, recorded at the collective's entry / exit
  double* d_part = nullptr;                       // [nranks] all-reduce staging (device)
  std::map<uint64_t, std::vector<tt_tensor>> reg; // tensor seq -> handle per rank
  std::mutex mu;
  std::condition_variable cv;
  int32_t arrived = 0;
  uint64_t gen = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == nranks) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  tt_tensor peer(const tt_tensor_s* t, int32_t rank) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = reg.find(t->seq);
    return it == reg.end() ? nullptr : it->second[rank];
  }
};
