/*
 * tt.h -- C ABI of the B200-native tiled block-sparse FP64 tensor contraction library (libtt.so).
 *
 * The library executes the data-parallel hot path of TAMM (arXiv 2201.01257): labelled tensor
 * set / addition / contraction over TiledIndexSpaces with block sparsity, on NVIDIA B200 (sm_100a).
 * Citations: P<n> = PAPER.md line n (/root/reference/PAPER.md, the paper's LaTeX source),
 * S<n> = SPEC.md line n, R<n> = reading n in DESIGN.md §3.
 *
 * Conventions (all entry points)
 *   - Every call returns tt_status: TT_OK (0) or a negative error code.  tt_last_error() returns a
 *     thread-local, NUL-terminated message describing the last failure on the calling thread.
 *   - Handles (tt_ctx, tt_is, tt_tis, tt_tensor) are opaque, created and destroyed by the library.
 *     They are immutable metadata with shallow-copy semantics (P212: "tensors in terms of handles ...
 *     any assignment done on tensor objects will be a shallow copy").
 *   - The library never allocates device memory on the execute path.  Tensor DATA is bound by the
 *     caller (e.g. a torch tensor, tt_tensor_bind); internal metadata (block maps, task lists, plans)
 *     and scratch (split-K and scalar partials) live in ONE caller-provided device workspace per
 *     context (tt_workspace_bind).  The caller keeps ownership of both; the library never frees them.
 *   - Execution is SPMD (P212, "single program multiple data"): with nranks > 1 every rank makes
 *     the same sequence of calls with identical metadata.  Compute calls are asynchronous on the
 *     context's CUDA stream; argument/validation errors are returned synchronously; CUDA and NCCL
 *     errors are returned by the call that observes them or by tt_sync.
 *   - Elements are IEEE FP64 (Tensor<double>, P130-132).
 *   - Labels are C strings with one character per dimension (e.g. "abij"); a character binds, by
 *     position, to that dimension's tiled index space (P145-159, Einstein notation).
 */
#ifndef TT_H_
#define TT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t tt_status;
enum {
  TT_OK = 0,
  TT_E_ARG = -1,        /* bad argument (NULL handle, out-of-range value, wrong length)              */
  TT_E_COVERAGE = -2,   /* tile sizes do not cover the index space exactly (P127; S83-87)            */
  TT_E_LABEL = -3,      /* label arity / dangling / repeated / batch label (S178, S380, S412)        */
  TT_E_TILING = -4,     /* matched labels on different tiled spaces (S413), or a tile straddles spin */
  TT_E_ZERO_BLOCK = -5, /* operation would write into a zero block (S208)                            */
  TT_E_UNBOUND = -6,    /* tensor has no storage bound, or the bound capacity is too small (S208)    */
  TT_E_OOM = -7,        /* internal metadata allocation failed                                       */
  TT_E_CUDA = -8,       /* CUDA runtime error (message in tt_last_error)                             */
  TT_E_NCCL = -9,       /* NCCL error                                                                */
  TT_E_STATE = -10,     /* call not valid in this state (e.g. device call on a host-only context)    */
  TT_E_UNSUPPORTED = -11,/* shape outside the supported envelope (e.g. order > TT_MAX_ORDER)         */
  TT_E_WORKSPACE = -12  /* no device workspace bound, or it cannot hold this call's metadata even     */
                        /* after evicting every unused cached plan (tt_workspace_bytes says how much) */
};

enum { TT_MAX_ORDER = 8 };          /* maximum tensor order                                        */
enum { TT_REPLICATED = -2 };        /* owner value: every rank holds the block                     */
enum { TT_SPLIT = -3 };             /* owner value: the block is owned by row-range parts          */
enum { TT_KIND_UNIFORM = 0, TT_KIND_INTEGER = 1 };   /* synthetic input kinds (tt_fill_synthetic)  */

typedef struct tt_ctx_s* tt_ctx;
typedef struct tt_is_s* tt_is;
typedef struct tt_tis_s* tt_tis;
typedef struct tt_tensor_s* tt_tensor;
typedef struct tt_sched_s* tt_sched;
typedef struct tt_sim_s* tt_sim;

/* Per-call statistics of the last set/add/contract/scalar call on a context (host-side counts). */
typedef struct {
  int64_t c_blocks;        /* output blocks computed by this rank                                  */
  int64_t tasks;           /* non-zero (A,B) tile pairs executed by this rank (contraction)        */
  int64_t work_items;      /* CTA work items launched                                              */
  double flops;            /* algorithmic FLOPs of this rank: sum over tasks of 2*prod(extents)    */
  double bytes;            /* compulsory HBM bytes of this rank (8*(A+B+(1+[beta!=0])*C elements)) */
  int64_t gathered_bytes;  /* bytes received from other ranks by the input-tile gather             */
  int64_t launches;        /* kernels launched by the call                                         */
  int32_t plan_cached;     /* 1 if the task list / partition / gather plan came from the cache     */
  int32_t kernel_variant;  /* contraction kernel tile variant used                  */
  int32_t producer;        /* operand staging of that kernel: 0 = cp.async, 1 = TMA; (T): 2 = pair  */
                           /* kernel, 3 = 2-CTA cluster with TMA multicast (tt_triples_energy)      */
  double aux_flops;        /* FLOPs spent building implicit operands (tt_contract_cholesky)         */
} tt_stats;

/* ------------------------------------------------------------------------------------------------
 * Execution context (P178-188: ExecutionContext{pg, &distribution, manager}).
 *   device      CUDA device ordinal, or -1 for a HOST-ONLY context (metadata, validation, host task
 *               lists and partitions only; every device call then returns TT_E_STATE).
 *   cuda_stream cudaStream_t the library launches on (NULL = legacy default stream); not owned.
 *   rank/nranks SPMD rank and size; 0 <= rank < nranks.
 *   nccl_id     pointer to a 128-byte ncclUniqueId (identical on all ranks) when nranks > 1 and
 *               device >= 0; otherwise NULL.  The library creates and owns the NCCL communicator.
 */
tt_status tt_ctx_create(int32_t device, void* cuda_stream, int32_t rank, int32_t nranks,
                        const void* nccl_id, tt_ctx* out);
tt_status tt_ctx_destroy(tt_ctx ctx);
/* Simulated ranks on ONE GPU (P212 SPMD with "access to the remote portions"; S506 rank
 * invariance): a group of nranks contexts on the same device, each created with tt_ctx_create_sim and
 * driven by its OWN host thread exactly as one process per GPU is (every rank makes the same call
 * sequence; each rank binds its own buffers).  Every multi-rank code path runs unchanged -- partitions,
 * owners, gather plans, row-split and compact storage -- except the transport: the input-tile gather
 * becomes one cudaMemcpyAsync (device to device, stream-ordered after the peer's producers via CUDA
 * events) per received run, read from the peer rank's buffer, and the scalar all-reduce a fixed
 * rank-order sum of the ranks' partials.  Each collective is a host barrier over the group, so a rank
 * that skips a collective the others make deadlocks (as NCCL would).  Tensors are matched across
 * ranks by creation order.  tt_sim_create allocates its small device staging here (device = the
 * group's GPU); destroy the group after all its contexts. */
tt_status tt_sim_create(int32_t device, int32_t nranks, tt_sim* out);
tt_status tt_sim_destroy(tt_sim sim);
/* Context of simulated rank `rank` of `sim` (stream: this rank's CUDA stream, not owned; use one
 * stream per rank). */
tt_status tt_ctx_create_sim(void* cuda_stream, int32_t rank, tt_sim sim, tt_ctx* out);
/* Writes a fresh ncclUniqueId (128 bytes) into out128 (rank 0 calls it and broadcasts the bytes). */
tt_status tt_nccl_unique_id(void* out128);
/* Record CUDA events around every kernel the library launches (for roofline timing). */
tt_status tt_ctx_set_profiling(tt_ctx ctx, int32_t enable);
/* Synchronises the context stream, then returns the summed event time (ms) and launch count of the
 * kernels whose name contains `kernel` ("" = all) since the last tt_profile_reset. */
tt_status tt_profile_read(tt_ctx ctx, const char* kernel, double* total_ms, int64_t* launches);
tt_status tt_profile_reset(tt_ctx ctx);
/* Statistics of the last compute call (see tt_stats). */
tt_status tt_last_stats(tt_ctx ctx, tt_stats* out);
/* Total kernels launched by the library on this context since creation. */
tt_status tt_launch_count(tt_ctx ctx, int64_t* out);
/* Blocks until all work queued on the context stream has finished; surfaces deferred errors. */
tt_status tt_sync(tt_ctx ctx);
/* Device workspace (P182-186: the ExecutionContext carries the memory manager).
 *   tt_workspace_bind(ctx, dev_ptr, bytes): binds caller-owned device memory (256-byte aligned,
 *     on the context's device; not owned, never freed by the library) from which every piece of
 *     library metadata and scratch of this context is carved.  Every device call needs a bound
 *     workspace (TT_E_WORKSPACE otherwise).  Re-binding (e.g. a larger buffer) first synchronises the
 *     device, drops every cached plan and every tensor's device metadata (rebuilt on next use); it
 *     is refused (TT_E_STATE) while a scheduler holds a captured graph of this context.  The old
 *     buffer may be freed by the caller once the call returns.  Cached plans that no running call
 *     holds are evicted least-recently-used when the workspace is full (after a device
 *     synchronisation: their regions may still be read by queued kernels).
 *   tt_workspace_bytes(ctx, &bytes): the size this context's workload needs: the high-water mark of
 *     live workspace bytes so far, raised to what a call that failed with TT_E_WORKSPACE needed
 *     (at least 1 MiB).  A call returns TT_E_WORKSPACE before it modifies any tensor, except
 *     tt_contract_cholesky, which builds its per-batch plans while it runs: give it room for all
 *     of them (tt_sched_* prepares every plan before the first launch).
 *   tt_workspace_info(ctx, &bound, &live, &high): bound size, bytes in use, high-water mark.
 *   tt_ctx_set_plan_limit(ctx, n): cached plans kept at most (default 16384; n >= 1); tt_ctx_clear_plans
 *     drops every cached plan that no running call or captured graph holds. */
tt_status tt_workspace_bind(tt_ctx ctx, void* dev_ptr, int64_t bytes);
tt_status tt_workspace_bytes(tt_ctx ctx, int64_t* bytes);
tt_status tt_workspace_info(tt_ctx ctx, int64_t* bound, int64_t* live, int64_t* high);
tt_status tt_ctx_set_plan_limit(tt_ctx ctx, int64_t max_plans);
tt_status tt_ctx_clear_plans(tt_ctx ctx);

/* ------------------------------------------------------------------------------------------------
 * IndexSpace (P116-122, Fig. 2: IndexSpace N{range(100)}).
 *   extent      number of indices (>= 1).
 *   n_ranges    0, or the number of ranges in begin_end; ranges must be ascending, non-empty and
 *               cover [0, extent) exactly (TT_E_COVERAGE otherwise).
 *   begin_end   2*n_ranges int64 [begin, end) pairs.
 *   spin        n_ranges values (+1 alpha, -1 beta) or NULL (no spin attribute).  P138: "encode spin
 *               information ... allocate these tensors using a block-sparse representation".
 * Tilings never straddle a range boundary (S39, reading R6).
 */
tt_status tt_is_create(int64_t extent, int32_t n_ranges, const int64_t* begin_end, const int8_t* spin,
                       tt_is* out);
tt_status tt_is_destroy(tt_is is);

/* TiledIndexSpace (P125-127): fixed tile size (remainder in the last tile of each range, R5) or
 * custom sizes with full coverage (TT_E_COVERAGE if they do not sum to the extent, TT_E_TILING if a
 * tile straddles a range boundary).  The tiled space keeps a reference to its index space. */
tt_status tt_tis_fixed(tt_is is, int64_t tile, tt_tis* out);
tt_status tt_tis_custom(tt_is is, int32_t n, const int64_t* sizes, tt_tis* out);
/* ntiles; offsets = ntiles+1 split points; tile_spin = per-tile spin (0 = none).  Pointers are owned
 * by the handle and valid until tt_tis_destroy. */
tt_status tt_tis_info(tt_tis tis, int32_t* ntiles, const int64_t** offsets, const int8_t** tile_spin);
tt_status tt_tis_destroy(tt_tis tis);
/* Sub-spaces (P116-122 named ranges "first"/"second"; P152 `tK("first").labels<3>()`; P159 "string-based
 * sub-spaces ... operations on different slices of the underlying allocated tensor").
 *   tt_tis_sub    the tiles of `parent` covering [begin, end); both ends must be tile boundaries of the
 *                 parent (TT_E_TILING otherwise).  Offsets are relative to begin, so a sub-space matches
 *                 (S413) any tiled space with the same tile sizes and spins.
 *   tt_tis_range  the sub-space of range `range` of the parent's index space (the paper's named
 *                 sub-range; names live in the caller, the index is the range's position).
 * The sub-space references its parent (keep it alive). */
tt_status tt_tis_sub(tt_tis parent, int64_t begin, int64_t end, tt_tis* out);
tt_status tt_tis_range(tt_tis parent, int32_t range, tt_tis* out);

/* ------------------------------------------------------------------------------------------------
 * Tensor<double> (P129-140): blocks indexed by the Cartesian product of the tiles of its dimensions
 * (row-major block grid; row-major elements inside a block, R9).  Storage is PACKED: only non-zero
 * blocks, in row-major block order, each block start rounded up to 2 doubles = 16 B (P210 third
 * scheme; R10).  Every rank uses the same packed layout; with nranks > 1 a rank holds valid data
 * only for the blocks it owns (default owners: round robin over non-zero blocks, P210).
 *   order       1..TT_MAX_ORDER (order 0 scalars are returned by tt_contract_scalar instead)
 *   dims        order tiled index spaces (referenced, not copied; keep them alive)
 *   nz          row-major u8 map over the block grid (1 = non-zero) or NULL = dense.
 * tt_tensor_create_spin derives nz from the spin rule of R7: a block is non-zero iff the sum of tile
 * spins over the dimensions in upper_mask equals the sum over lower_mask (bit d = dimension d).
 */
tt_status tt_tensor_create(tt_ctx ctx, int32_t order, const tt_tis* dims, const uint8_t* nz,
                           tt_tensor* out);
tt_status tt_tensor_create_spin(tt_ctx ctx, int32_t order, const tt_tis* dims, uint32_t upper_mask,
                                uint32_t lower_mask, tt_tensor* out);
tt_status tt_tensor_info(tt_tensor t, int32_t* order, int64_t* nblocks, int64_t* nnz_blocks);
/* packed_elems = elements the bound buffer must hold; blk_off[nblocks] (-1 = zero block);
 * owner[nblocks] (-1 = zero block, TT_REPLICATED, or a rank); nz[nblocks].  Owned by the handle.
 * These maps are the frozen layout contract compared bit-exactly with the oracle. */
tt_status tt_tensor_layout(tt_tensor t, int64_t* packed_elems, const int64_t** blk_off,
                           const int32_t** owner, const uint8_t** nz);
/* Replace the owner map (nblocks entries; zero blocks ignored; values in [0,nranks) or
 * TT_REPLICATED).  Must be identical on every rank. */
tt_status tt_tensor_set_owner(tt_tensor t, const int32_t* owner);
/* Row-range ownership (SURVEY §8(e) "block splitting", owner-computes at a finer grain than a block):
 * part i is rows [lo[i], hi[i]) of the dimension-0 tile of block blk[i], owned by rank owner[i].  The
 * parts of a block must tile its dimension-0 range in order; listed blocks get owner TT_SPLIT (one
 * part covering the whole tile = an ordinary owner); unlisted blocks keep their owner.  Because
 * dimension 0 is outermost, a part is a contiguous element range of the packed block.  Must be
 * identical on every rank. */
tt_status tt_tensor_set_parts(tt_tensor t, int64_t n, const int64_t* blk, const int32_t* lo,
                              const int32_t* hi, const int32_t* owner);
/* The parts of all split blocks (arrays owned by the handle, valid until the next ownership change). */
tt_status tt_tensor_parts(tt_tensor t, int64_t* n, const int64_t** blk, const int32_t** lo,
                          const int32_t** hi, const int32_t** owner);
/* Compact storage (memory for 180 GB per GPU at configs[4] scale): with on != 0 the bound buffer
 * holds only the element ranges THIS rank holds (its owned blocks and row parts, and replicated
 * blocks): per non-zero block the span from its first to its last held element, packed in block
 * order, each block base 16-B aligned.  Storage offsets are recomputed on every ownership change
 * (set_owner / set_parts / partitions).  A compact tensor may be the output of any operation and an
 * input whose reads are all local; an operation that would gather remote pieces INTO it fails with
 * TT_E_UNSUPPORTED (on every rank alike).  upload/download move the storage buffer.  Must be
 * identical on every rank.  Default off (storage = the global packed layout). */
tt_status tt_tensor_set_compact(tt_tensor t, int32_t on);
/* Sliced view (P152, P159): a tensor whose dimension d is dims[d] = the tensor's own tiled space or a
 * sub-space of it (tt_tis_sub / tt_tis_range of exactly T's dims[d]; TT_E_TILING otherwise).  The view's
 * blocks ARE the parent's blocks at the shifted tile coordinates: same storage (the parent's current
 * binding is used at every call), same packed offsets and owners, no copy.  A view can be an operand or
 * the output of every operation; reads and writes go to the parent's memory.  Its block map, offsets
 * and owners are captured at creation, so while a view of T exists, ownership / compact / partition
 * changes of T return TT_E_STATE (destroy the views, change T, re-create them); views of compact or
 * row-split tensors, views of views, and ownership / compact changes on a view are TT_E_UNSUPPORTED.  tt_fill_synthetic on a view uses the view's own global indices.  Destroy the view
 * before its parent. */
tt_status tt_tensor_view(tt_tensor T, const tt_tis* dims, tt_tensor* out);
/* Storage size in doubles (what tt_tensor_bind needs) and the per-block storage offsets (nblocks
 * entries; -1 = not stored on this rank; block base, i.e. element e of block b is at off[b] + e).
 * Without compact storage these equal packed_elems / blk_off of tt_tensor_layout. */
tt_status tt_tensor_storage(tt_tensor t, int64_t* storage_elems, const int64_t** storage_off);
/* Bind caller-owned DEVICE memory of capacity_elems doubles (>= the storage size: packed_elems, or
 * tt_tensor_storage's size when compact; 16-B aligned). */
tt_status tt_tensor_bind(tt_tensor t, void* dev_ptr, int64_t capacity_elems);
/* Host <-> device copies of the whole storage buffer on the context stream (asynchronous when the
 * host memory is pinned).  host holds the storage size in doubles (packed_elems unless compact).  These are the end-to-end entry points
 * for callers whose data lives in host memory. */
tt_status tt_tensor_upload(tt_ctx ctx, tt_tensor t, const double* host);
tt_status tt_tensor_download(tt_ctx ctx, tt_tensor t, double* host);
tt_status tt_tensor_destroy(tt_tensor t);

/* Seeded synthetic input (not part of the method): every element of every non-zero
 * block this rank holds is set to the counter-based generator value at its GLOBAL row-major index g:
 *   h = splitmix64(seed ^ (tag * 0x9E3779B97F4A7C15) ^ g)
 *   kind UNIFORM: (h >> 11) * 2^-53 * 2 - 1;   kind INTEGER: (h mod 5) - 2.
 * Identical to synthetic/__init__.py (checked bit-exactly by tests). */
tt_status tt_fill_synthetic(tt_ctx ctx, tt_tensor t, uint64_t seed, uint32_t tag, int32_t kind);

/* ------------------------------------------------------------------------------------------------
 * Operations (P170-174, grammar rules 5-7; "=" is beta = 0 and never reads C, "+=" is beta = 1,
 * general beta per BASELINE north_star; R3, R4).  Only non-zero C blocks owned by this rank (or
 * replicated) are written; zero input blocks read as zeros (S216); no contribution is computed for
 * a zero C block (R8).
 *
 * tt_set       C = alpha                                      (P172, rule 5)
 * tt_add       C(c_lbl) = beta*C + alpha*A(a_lbl)             (P173, rule 6: a_lbl is a permutation
 *                                                              of c_lbl, same tiled spaces)
 * tt_contract  C(c_lbl) = beta*C + alpha*sum A(a_lbl)*B(b_lbl) (P174, rule 7): contracted labels are
 *              the labels in both A and B and not in C; every C label appears in exactly one of A, B;
 *              no label repeats within an operand; a label in all three is rejected (TT_E_LABEL);
 *              matched labels must use the same tt_tis (TT_E_TILING).
 *              Each non-zero C block is the sum over the non-zero (A,B) tile pairs of the task list
 *              (tt_task_list) of a dense FP64 contraction, executed by the DMMA kernel with the
 *              index permutation folded into the operand staging.  With nranks > 1
 *              the rank computes the C blocks it owns and first receives, over NCCL, exactly the A/B
 *              blocks its tasks read but does not own (P212 "access to the remote portions").
 *              Kernel tile variant: a cost model, refined by measured autotuning for plans of
 *              >= 5e10 FLOPs (the first two calls time the model's choice and its runner-up; later
 *              calls use the faster; the variants give identical bits; TT_AUTOTUNE=0 disables it,
 *              TT_FORCE_VARIANT=v forces one).
 * tt_contract_scalar  *result = alpha * sum_x A(x)*B(x) over all labels (order-0 result such as the
 *              CC energy, P534-536), summed over ranks with an NCCL all-reduce; *result is a HOST
 *              pointer and the call synchronises the stream.  With nranks > 1 each rank sums the A
 *              blocks it owns (replicated blocks: rank 0).
 */
tt_status tt_set(tt_ctx ctx, tt_tensor C, double alpha);
tt_status tt_add(tt_ctx ctx, tt_tensor C, const char* c_lbl, double beta, double alpha, tt_tensor A,
                 const char* a_lbl);
tt_status tt_contract(tt_ctx ctx, tt_tensor C, const char* c_lbl, double beta, double alpha,
                      tt_tensor A, const char* a_lbl, tt_tensor B, const char* b_lbl);
/* Prefetch of the input gather of a later tt_contract with the same arguments (SURVEY §8(e) "gathers run on
 * a comm stream ... overlapped with compute"): the NCCL send/recv of exactly the input ranges this rank's
 * tasks read but does not hold is issued now on the context's communication stream, after everything
 * already issued on the context stream (so earlier kernels that read those ranges are not overwritten);
 * the next tt_contract of this plan (same tensors, labels, beta != 0 or == 0) waits for it instead of
 * gathering, so its kernel starts as soon as the data is there and the transfer overlaps whatever runs on
 * the context stream in between (e.g. the previous contraction's kernel).  Gathers that are not prefetched
 * wait for pending prefetched ones (one communicator is never used by two streams at once).  SPMD: every
 * rank issues the same prefetch / contract sequence.  No-op with nranks == 1.  TT_E_STATE if this
 * contraction is already prefetched and not yet executed. */
tt_status tt_contract_prefetch(tt_ctx ctx, tt_tensor C, const char* c_lbl, double beta, tt_tensor A,
                               const char* a_lbl, tt_tensor B, const char* b_lbl);

/* End-to-end contraction from HOST memory (P178-188 execution on host-resident data; the caller's
 * pinned buffers give full overlap): hA, hB, hC are host copies of the packed STORAGE of A, B, C (the
 * same layout as tt_tensor_upload; NULL = that operand is already resident on the device, no copy).
 * c_flags: TT_HOST_C_IN uploads C first (needed when beta != 0 and C is not resident), TT_HOST_C_OUT
 * downloads C after the contraction.  Device buffers of A, B, C must be bound (copy destinations).
 * With A's dim 0 labelled like C's dim 0 (same tiled space; no views, A != B, C not compact) and, with
 * several ranks, A's rows local to this rank's C rows (no gather of A; B's remote blocks are gathered
 * first), the call is PIPELINED over the blocks / row parts this rank holds: per chunk x of C (its blocks sharing the dim-0 tile, or the (dim-0,
 * dim-1) tile pair when dim 0 has fewer than 16 tiles and A's dim 1 carries C's dim-1 label), A's blocks
 * with the same leading coordinates (one packed range) are copied host->device on the context's copy
 * stream while chunk x-1 contracts, and C's rows of chunk x go back while chunk x+1 contracts; each chunk
 * is computed with the same per-element k order as the whole contraction, so the result is bitwise that
 * of upload + tt_contract + download.  Otherwise every
 * rank copies the ranges it holds (owned blocks / row parts, replicated blocks), runs tt_contract (the
 * gathers fetch the rest over NVLink) and copies back its own C ranges.  Asynchronous on the context
 * stream like tt_contract: the host buffers must stay valid until tt_sync.  Errors as tt_contract. */
enum { TT_HOST_C_IN = 1, TT_HOST_C_OUT = 2 };
tt_status tt_contract_host(tt_ctx ctx, tt_tensor C, const char* c_lbl, double beta, double alpha, tt_tensor A,
                           const char* a_lbl, tt_tensor B, const char* b_lbl, const double* hA, const double* hB,
                           double* hC, int32_t c_flags);
tt_status tt_contract_scalar(tt_ctx ctx, double alpha, tt_tensor A, const char* a_lbl, tt_tensor B,
                             const char* b_lbl, double* result);

/* Three-operand contraction through an intermediate (PAPER Eqs. cc9-cc11, P293-311):
 *   C(c_lbl) = beta*C + alpha * sum A(a_lbl) * B(b_lbl) * D(d_lbl)
 * e.g. cc9 "1/4 v^{ef}_{mn} t^{ij}_{ef} t^{mn}_{ab}": C = R "abij", A = v "efmn", B = t "efij", D = t "abmn",
 * alpha = 1/4.  Every label must appear in exactly two of C, A, B, D (TT_E_LABEL).  The three pairings
 * (A*B)*D, (A*D)*B, (B*D)*A are costed on the block maps: the intermediate I of a pair (X, Y) carries the
 * labels of X then Y that survive (appear in the third operand or C), on their tiled spaces, and its
 * block map is the set of blocks that receive at least one non-zero pair; the cost is the FLOPs
 * (2*m*n*k per task, as tt_task_list) of I = X*Y plus C += I*Z.  The cheapest pairing (ties: the first in
 * the order above; reading R26) runs as two tt_contract calls (I = 1*X*Y with beta 0, then
 * C = beta*C + alpha*I*Z), I stored in the caller's workspace.
 *   workspace  device memory of ws_elems doubles >= info->ws_elems (I's packed size), or NULL to
 *              return only the plan (info) without computing.
 *   info       (may be NULL) pair = 0/1/2 in the order above; i_lbl = the intermediate's labels;
 *              flops[p] = factorized FLOPs of pairing p (-1: intermediate order > TT_MAX_ORDER);
 *              naive_macs = multiply-adds of the unfactorized loop (one product per combination of
 *              all label values whose C, A, B, D blocks are non-zero; n_o^4 n_u^4 for dense cc9;
 *              -1 if the label tile grid exceeds 5e7 tuples); ws_elems = intermediate size in doubles.
 * With nranks > 1 I is owned round robin (P210) and the second contraction gathers what it reads.
 * tt_stats after the call = the sum over both contractions. */
typedef struct {
  int32_t pair;
  char i_lbl[TT_MAX_ORDER + 1];
  double flops[3];
  double naive_macs;
  int64_t ws_elems;
} tt_contract3_info;
tt_status tt_contract3(tt_ctx ctx, tt_tensor C, const char* c_lbl, double beta, double alpha,
                       tt_tensor A, const char* a_lbl, tt_tensor B, const char* b_lbl, tt_tensor D,
                       const char* d_lbl, void* workspace, int64_t ws_elems, tt_contract3_info* info);

/* Perturbative triples correction (T) (PAPER Eqs. cc13, cc14, tensort, abt, tensort2,
 * P343-413):
 *   E(T) = sum_{i<j<k, a<b<c} (W + V1) * W / (e_i + e_j + e_k - e_a - e_b - e_c)          (Eq. cc14, R28)
 *   W  = Eq. tensort: 9 terms v^{xy}_{mp} t^{mz}_{qr} summed over occupied m (A of Eq. abt) and 9 terms
 *        v^{ex}_{pq} t^{yz}_{er} summed over virtual e (B); the sixth term with "-" (reading R27),
 *   V1 = Eq. tensort2: the nine v^{xy}_{pq} t^z_r products.
 * Inputs (real amplitudes and integrals; storage conventions of oracle/triples.py):
 *   T1     t^i_a       as T1(a,i)        dims (V, O)      -- V = T1's dim 0 tiling, O = its dim 1 tiling
 *   T2     t^{ij}_{ab} as T2(a,b,i,j)    dims (V, V, O, O)
 *   Vooov  v^{ij}_{ma} as Vooov(i,j,m,a) dims (O, O, O, V)
 *   Vvovv  v^{ei}_{ab} as Vvovv(e,i,a,b) dims (V, O, V, V)
 *   Voovv  v^{ij}_{ab} as Voovv(i,j,a,b) dims (O, O, V, V)
 *   every dim must be T1's tiled-space object itself (TT_E_TILING); zero blocks read as 0, and every
 *   non-zero block must obey the spin rule the kernel prunes by (sum of the tile spins of dims {0,1}
 *   = that of dims {2,3}; T1: s_a = s_i) -- on spaces without spin any map passes, on alpha/beta
 *   spaces a block outside the R7 spin map is TT_E_UNSUPPORTED; virtual ranges must have even sizes (TT_E_UNSUPPORTED); eps_o[n_o], eps_v[n_v]: DEVICE arrays
 *   of orbital energies (global index order).
 * Execution: the inputs are copied into dense permuted layouts in the workspace; then one fused kernel
 * CTA per unit = (occupied triple i<j<k, triple of 16-wide virtual boxes b_a <= b_b <= b_c) forms the
 * unit's W in shared memory as W(a,b,c) = G(a;b,c) - G(b;a,c) + G(c;a,b) -- the 18 terms regrouped into
 * three DMMA GEMMs with K = 3 n_o + 3 n_v -- and reduces (W + V1) W / D over a<b<c into one partial per
 * unit; a fixed-order sum gives E (deterministic).  Units whose box spins and occupied spins differ in
 * sum are skipped (W = 0 under the spin maps of R7).  With nranks > 1 the inputs may have any whole-block
 * owners (not compact): every rank first gathers the blocks it does not hold into the inputs' own
 * storage (the kernel reads all of them), the units are split into contiguous ranges of equal modelled
 * cost (cost_* below) and E
 * is all-reduced (NCCL).
 * energy: HOST pointer; the call synchronises the stream.
 *   workspace  device memory of ws_elems doubles >= info->ws_elems (dense copies + one partial per
 *              unit), or NULL to return only info.
 *   info       (may be NULL) w_blocks_total / w_blocks = units in total / on this rank; batches = 1;
 *              flops_alg = FLOPs of the defined sums over the restricted elements (a<b<c, i<j<k,
 *              spin-allowed) of this rank: 2 per non-zero product of the 18 terms (18 (n_o + n_v) per
 *              element without spin; only the spin-allowed half of each m / e sum with alpha/beta
 *              spaces); flops_exec = FLOPs of the DMMAs the default kernel issues on this rank (only the
 *              8x8 output fragments holding a needed element, 8-row stages per m / e segment; with
 *              alpha/beta spaces only the spin-allowed half of each m / e sum is run);
 *              ws_elems = workspace needed;
 *              cost_rank / cost_total / cost_max_unit = modelled cost (needed fragments x stages over the
 *              three GEMMs + a fixed 448 per unit) of this rank's units / all units / the costliest unit:
 *              the split gives every rank cost_total / nranks within one unit's cost. */
typedef struct {
  int64_t w_blocks_total, w_blocks, batches;
  double flops_alg, flops_exec;
  int64_t ws_elems;
  double cost_rank, cost_total, cost_max_unit;
} tt_triples_info;
tt_status tt_triples_energy(tt_ctx ctx, tt_tensor T1, tt_tensor T2, tt_tensor Vooov, tt_tensor Vvovv,
                            tt_tensor Voovv, const double* eps_o, const double* eps_v, void* workspace,
                            int64_t ws_elems, double* energy, tt_triples_info* info);

/* Contraction with an IMPLICIT Cholesky-factored operand (PAPER Eq. cc12,
 * P312-318, the paper's CD-CCSD P325/P463):
 *   C(c_lbl) = beta*C + alpha * sum V(v_lbl) * B(b_lbl),
 *   V(p,q,r,s) = sum_L X(p,r,L) X(q,s,L) - X(p,s,L) X(q,r,L)     (v_lbl = "pqrs"; formula as printed, R19)
 * V is never stored.  Since the exchange term is the Coulomb term W(p,q,r,s) = sum_L X(p,r,L)X(q,s,L)
 * with r,s swapped, the call evaluates the identical sum W * (B - B(r<->s)): Bm = B - B(r<->s) is formed
 * once in the workspace, then the rank's C parts are processed in batches of (p,q) tile rows whose W
 * blocks are built by the DMMA contraction kernel (over L) into the rest of the workspace and consumed
 * by the contraction restricted to the batch.  workspace: caller-owned device memory of ws_elems
 * doubles >= B's packed size (rounded up to 32) + one (p,q) row of W.  Ladder form only: p, q free
 * labels of C, r, s contracted with B; X(p,r,L) order 3 with dims 0 and 1 on the tiled space of p,q,r,s.
 * B is all-gathered once per call; with nranks > 1 X may have any owners (not compact): the blocks a rank
 * does not hold are gathered once per call (every rank builds W from all of X).
 * tt_stats.flops = algorithmic FLOPs of the defined contraction over V's block map (non-zero iff the
 * Coulomb or the exchange term conserves spin pairwise); aux_flops = FLOPs executed (W build + consume). */
tt_status tt_contract_cholesky(tt_ctx ctx, tt_tensor C, const char* c_lbl, double beta, double alpha,
                               tt_tensor X, const char* v_lbl, tt_tensor B, const char* b_lbl,
                               void* workspace, int64_t ws_elems);

/* ------------------------------------------------------------------------------------------------
 * Task list (canonical order, R11): for each non-zero C block in row-major order (all of them, not
 * only owned ones), each contracted-tile tuple in row-major order with the contracted labels in order
 * of first appearance in A: a task (A block id, B block id) iff both blocks are non-zero.
 *   where       0 = host enumerator, 1 = the device builder (count -> scan -> fill) copied back.
 *   cblk        [n_cblocks] non-zero C block ids;  ptr [n_cblocks+1] CSR offsets into a_blk/b_blk.
 *   cost        [n_cblocks] FLOPs per C block = sum over its tasks of 2*prod(extents of all labels).
 * Two-call pattern: pass NULL arrays (cap ignored) to get n_cblocks / n_tasks; then arrays of that
 * size (cap = capacity of a_blk/b_blk) -- TT_E_ARG if too small.
 */
tt_status tt_task_list(tt_ctx ctx, tt_tensor C, const char* c_lbl, tt_tensor A, const char* a_lbl,
                       tt_tensor B, const char* b_lbl, int32_t where, int64_t* cblk, int64_t* ptr,
                       int64_t* a_blk, int64_t* b_blk, int64_t* cost, int64_t cap,
                       int64_t* n_cblocks, int64_t* n_tasks);

/* LPT owner partition of C's non-zero blocks over the context's nranks (R24): units sorted by
 * (cost desc, smallest block id asc), each to the least-loaded rank, ties to the lowest rank.
 *   group_mask  0: every non-zero C block is a unit.  Otherwise bit d set = C dimension d is a
 *               grouping dimension: blocks with equal tile coordinates on all grouping dimensions
 *               form one unit (e.g. the (a,b) rows of R(a,b,i,j) with mask 0b0011, so that the
 *               V(a,b,c,d) rows each rank reads are its own).  Unit cost = sum of block costs.
 * Writes owner[nblocks of C] (-1 for zero blocks).  Does not modify C (use tt_tensor_set_owner). */
tt_status tt_partition_lpt(tt_ctx ctx, tt_tensor C, const char* c_lbl, tt_tensor A, const char* a_lbl,
                           tt_tensor B, const char* b_lbl, uint32_t group_mask, int32_t* owner);

/* Balanced owner-computes partition with row splitting (reading R24): units (blocks,
 * or groups of blocks per group_mask, which must then include dimension 0) are ordered by (cost desc,
 * smallest block id asc) and laid along a cost axis; rank r gets [floor(r*W/P), floor((r+1)*W/P)) of
 * it, and a unit that straddles a boundary is cut at the nearest row of its dimension-0 tile (round
 * half up).  Balance is exact to one row; at most P-1 units are split.  Writes C's owners / parts
 * (as tt_tensor_set_owner + tt_tensor_set_parts). */
tt_status tt_partition_split(tt_ctx ctx, tt_tensor C, const char* c_lbl, tt_tensor A, const char* a_lbl,
                             tt_tensor B, const char* b_lbl, uint32_t group_mask);

/* As tt_partition_split with caller-supplied costs instead of a contraction's task list, for
 * operations whose work is not one contraction's (e.g. the implicit Cholesky evaluation, whose
 * work per row is its W formation plus the GEMMs over W's block map, reading R19b).
 *   cost  [number of non-zero C blocks] non-negative cost of each non-zero C block, in block-id
 *         order (host pointer, read only).  TT_E_ARG on NULL or a negative cost. */
tt_status tt_partition_split_cost(tt_ctx ctx, tt_tensor C, const int64_t* cost, uint32_t group_mask);
/* R24b on the executed cost of the implicit-operand ladder C(..p..q..) += V(p,q,r,s) B(..r..s..)
 * (tt_contract_cholesky, Eq. cc12; same arguments and checks): per non-zero C block, the GEMM FLOPs of
 * its tasks over W's block map (W(pqrs) = sum_L X(prL) X(qsL), map from X's block map, R19b) plus the
 * W formation of its (p_t, q_t) row, 2 N_L |p||q| sum over W's (r_t, s_t) blocks of |r||s|, shared
 * evenly (integer division) by the row's non-zero C blocks; then as tt_partition_split_cost. */
tt_status tt_partition_split_cholesky(tt_ctx ctx, tt_tensor C, const char* c_lbl, tt_tensor X, const char* v_lbl,
                                      tt_tensor B, const char* b_lbl, uint32_t group_mask);

/* Input-tile gather plan of this rank for tt_contract (host metadata; for tests and reports).
 * recv[5*i .. 5*i+4] = (operand 0=A/1=B, block id, source rank, e0, e1): element range [e0, e1) of
 * the block this rank receives (whole blocks, or rows of row-split parts);
 * send[5*i .. 5*i+4] = (operand, block id, destination rank, e0, e1).  Two-call pattern as
 * tt_task_list. */
tt_status tt_gather_plan(tt_ctx ctx, tt_tensor C, const char* c_lbl, tt_tensor A, const char* a_lbl,
                         tt_tensor B, const char* b_lbl, int64_t* recv, int64_t* n_recv,
                         int64_t* send, int64_t* n_send, int64_t cap);

/* ------------------------------------------------------------------------------------------------
 * Scheduler (P178, P191-199, P215: "Scheduler sch{&ec}; sch(op)(op)...execute()").  Operations are
 * queued (arguments as the immediate calls; tensors and host result pointers must stay valid until
 * tt_sched_execute returns) and executed in LEVELS (reading R25): two ops conflict when they share a
 * tensor and one of them writes it (a "+=" / beta != 0 update reads and writes its output); the level
 * of an op is 1 + the largest level of the earlier ops it conflicts with (0 if none).  Each level's
 * ops run concurrently on the scheduler's `nstreams` CUDA streams, forked from and joined back into
 * the context stream (one synchronisation point per level); with nranks > 1 they run in queue order
 * on the context stream (every rank then issues its NCCL calls in the same order).  execute clears
 * the queue.  A host-only context can queue and levelize but not execute (TT_E_STATE). */
tt_status tt_sched_create(tt_ctx ctx, int32_t nstreams, tt_sched* out);
tt_status tt_sched_destroy(tt_sched s);
tt_status tt_sched_set(tt_sched s, tt_tensor C, double alpha);
tt_status tt_sched_add(tt_sched s, tt_tensor C, const char* c_lbl, double beta, double alpha, tt_tensor A,
                       const char* a_lbl);
tt_status tt_sched_contract(tt_sched s, tt_tensor C, const char* c_lbl, double beta, double alpha,
                            tt_tensor A, const char* a_lbl, tt_tensor B, const char* b_lbl);
tt_status tt_sched_contract_cholesky(tt_sched s, tt_tensor C, const char* c_lbl, double beta, double alpha,
                                     tt_tensor X, const char* v_lbl, tt_tensor B, const char* b_lbl,
                                     void* workspace, int64_t ws_elems);
tt_status tt_sched_scalar(tt_sched s, double alpha, tt_tensor A, const char* a_lbl, tt_tensor B,
                          const char* b_lbl, double* result);
/* level[nops] of every queued op (NULL to query only), nops, number of levels. */
tt_status tt_sched_levels(tt_sched s, int32_t* level, int64_t* nops, int32_t* nlevels);
tt_status tt_sched_execute(tt_sched s);
/* CUDA graph of the queue (iterative methods replay the same operations; launch-bound small problems
 * pay one graph launch instead of per-op host work and launches): capture builds every plan first
 * (outside the capture), then records the levels -- streams, fork/join events, NCCL calls -- into a
 * graph; the queue is kept.  replay launches the graph on the context stream; if the queue has scalar
 * ops their results are copied to the host pointers given at queue time (the call then synchronises).
 * A later tt_sched_execute clears the queue and the graph. */
tt_status tt_sched_capture(tt_sched s);
tt_status tt_sched_replay(tt_sched s);
tt_status tt_sched_stats(tt_sched s, int64_t* queued, int64_t* levels_executed);

const char* tt_last_error(void);
int32_t tt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TT_H_ */
