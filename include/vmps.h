/*
 * vmps.h -- C ABI of the B200-native (sm_100a) Virtual-Memory Powersort hot
 * path (arXiv 2605.27147).  libvmps.so exports exactly the functions below.
 *
 * The operation.  vmps_sort_keys / vmps_sort_pairs compute the stable sort of
 * n items (key, optional u32 payload) in place -- Alg. 1 "Abstract Powersort"
 * sorts input[0,n) in place -- by merging the
 * array's natural runs along the Powersort merge tree:
 *   - runs: ExtractRun with minrun extension by insertion sort
 *     ("l = ceil(l/2) until l < 64"); strictly descending runs are
 *     reversed (BASELINE.json north_star; reading R3);
 *   - node powers (Theorem): the power of the boundary between runs
 *     [i,j) and [j,k) is the least p with an integer c such that
 *     (i+j)/2n < c 2^-p <= (j+k)/2n;
 *   - merges: every merge is stable, ties taken from the left run (Alg. 2,
 *     P:657 "a[x_a] <= b[x_b]").
 * The output is the unique stable sort (F1), bit-identical to the
 * oracle.  vmps_merge_plan reports Alg. 1's merge sequence.
 *
 * Conventions (all functions):
 *   - Pointers are DEVICE pointers unless the name starts with h_ (host).
 *   - Key order: VMPS_KEY_U32 / VMPS_KEY_U64 unsigned; VMPS_KEY_F32 is a
 *     total order in which -0.0 precedes +0.0, every NaN is greater than every
 *     non-NaN and all NaNs compare equal (stable among themselves); output
 *     keys keep their bit patterns (reading R5).
 *   - n <= VMPS_MAX_N = 2^32 - 2^16 per call (32-bit positions inside the
 *     library, with headroom for position + tile / minrun sums); larger n
 *     returns VMPS_ERR_INVALID_ARG.
 *   - Ownership: keys, vals and ws are caller-owned and must stay valid until
 *     the work enqueued on `stream` completes.  The library allocates no
 *     device memory; it uses the caller's workspace (size from
 *     vmps_workspace_bytes, 256-byte aligned).
 *   - Asynchrony: all device work is enqueued on `stream` (0 = legacy
 *     default stream).  Functions return after enqueueing, except that a
 *     non-NULL h_stats / h_num_runs synchronises `stream` to read results.
 *   - Errors: arguments are validated before anything is enqueued.
 *       VMPS_ERR_INVALID_ARG  NULL pointer with n > 1, unknown key type,
 *                             n > VMPS_MAX_N, misaligned pointer (keys/vals must be
 *                             16-byte aligned), cap_runs too small (the needed
 *                             count is still written to *h_num_runs);
 *       VMPS_ERR_BUDGET       ws_bytes smaller than vmps_workspace_bytes(), or
 *                             scratch_elems below the bounded mode's minimum;
 *       VMPS_ERR_CUDA         a CUDA launch/runtime error (detail:
 *                             vmps_last_error());
 *     n <= 1 is a no-op returning VMPS_OK.  There is no CPU fallback.
 *   - Thread safety: calls on different streams with different workspaces may
 *     run concurrently; the vmps_test_* hooks are process-global and are not.
 */
#ifndef VMPS_H
#define VMPS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VMPS_MAX_N 4294901760ull /* 2^32 - 2^16: the largest n of one call */

typedef enum { VMPS_KEY_U32 = 0, VMPS_KEY_U64 = 1, VMPS_KEY_F32 = 2 } vmps_key_t;

typedef enum {
  VMPS_OK = 0,
  VMPS_ERR_INVALID_ARG = 1,
  VMPS_ERR_ALLOC = 2,
  VMPS_ERR_BUDGET = 3,
  VMPS_ERR_CUDA = 4,
  VMPS_ERR_NCCL = 5,
  VMPS_ERR_INTERNAL = 6
} vmps_status_t;

/* scratch_elems value selecting the unbounded (ping-pong) mode */
#define VMPS_SCRATCH_UNBOUNDED (-1LL)

/* Run kinds reported by vmps_merge_plan (bit flags). */
#define VMPS_RUN_ASC 0u
#define VMPS_RUN_DESC 1u /* strictly descending, reversed */
#define VMPS_RUN_EXT 2u  /* shorter than minrun, extended by insertion sort */

/* Statistics; filled only when a non-NULL h_stats is passed (synchronises). */
typedef struct {
  uint64_t n;
  uint64_t runs;           /* r: runs after ExtractRun */
  uint64_t merges;         /* r - 1 */
  uint64_t merge_cost_M;   /* sum of merge input lengths */
  uint64_t fused_M;        /* part of M executed inside block-local sorts */
  uint64_t reversed_elems; /* elements of strictly descending runs */
  uint64_t extended_runs;  /* runs extended to minrun */
  uint32_t max_power;      /* largest node power */
  uint32_t levels_executed;/* merge levels with at least one HBM merge */
  uint32_t minrun;
  uint32_t block_elems;    /* bounded mode: block size P_blk (0 if unbounded) */
  uint64_t rounds;         /* bounded mode: level passes that moved data (0 if unbounded) */
  uint64_t peak_extra_device_bytes; /* workspace bytes actually used */
  uint64_t scratch_bytes;  /* element scratch part of it */
  uint64_t metadata_bytes; /* plan / table / relocation metadata part of it */
  uint64_t hbm_merge_elems;/* elements written by the HBM merge passes (sum of the
                              materialized non-fused node sizes; = M - fused_M with
                              one level per pass, about half of it with two) */
} vmps_stats_t;

/* One merge of the plan: [i,j) with [j,k) at node power `power`; `order` is
 * the rank in Alg. 1's execution order (records are written in that order). */
typedef struct {
  uint64_t i, j, k;
  uint32_t power;
  uint32_t order;
} vmps_merge_rec_t;

/* Workspace size for a sort (has_vals: payload present) or, with
 * has_vals = -1, for vmps_merge_plan.  scratch_elems as in vmps_sort_*. */
vmps_status_t vmps_workspace_bytes(uint64_t n, vmps_key_t kt, int has_vals,
                                   int64_t scratch_elems, size_t* h_bytes);

/* Stable in-place sort of keys[0,n) (layout: contiguous array of the key
 * type).  scratch_elems: VMPS_SCRATCH_UNBOUNDED, or a cap on element scratch
 * (bounded mode: the output is identical; BASELINE.json north_star (4); the
 * paper's VM Powersort).  Bounded mode: one dataflow pass per
 * merge level through a block table (free blocks reused as soon as their
 * elements are consumed), then the Copy into physical order; above two cells
 * of 2^23 elements the plan is processed in dyadic cells of the run
 * midpoints so that metadata is O(cell / minrun + n / P) and the
 * executed merges are still exactly Alg. 1's.  The bounded mode synchronises
 * `stream` (per cell and at the end). */
vmps_status_t vmps_sort_keys(void* keys, uint64_t n, vmps_key_t kt, int64_t scratch_elems,
                             void* ws, size_t ws_bytes, void* stream, vmps_stats_t* h_stats);

/* As vmps_sort_keys; vals[0,n) (u32) is permuted with its keys. */
vmps_status_t vmps_sort_pairs(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt,
                              int64_t scratch_elems, void* ws, size_t ws_bytes, void* stream,
                              vmps_stats_t* h_stats);

/* Host-buffer entry points (end-to-end path): h_keys[0,n) (and h_vals) live
 * in host memory (pinned for asynchronous copies; pageable works but the
 * copies then block the calling thread).  Enqueued on `stream`: copy to the
 * caller's device buffers d_keys / d_vals (n elements each, 16-byte
 * aligned), the device sort exactly as vmps_sort_keys / vmps_sort_pairs, and
 * the copy of the sorted result to h_keys_out / h_vals_out (host; NULL =
 * in place into h_keys / h_vals).  Returns after enqueueing (h_stats != NULL
 * synchronises and fills only h_stats->n); the host output holds the result
 * once `stream` completes.  Calls on different streams with their own device
 * buffers and workspaces overlap one batch's copies with another's sort.
 * Errors as vmps_sort_*, validated before anything is enqueued; NULL input
 * or device pointers with n > 1 are VMPS_ERR_INVALID_ARG. */
vmps_status_t vmps_sort_keys_host(const void* h_keys, void* h_keys_out, uint64_t n, vmps_key_t kt,
                                  int64_t scratch_elems, void* d_keys, void* ws, size_t ws_bytes,
                                  void* stream, vmps_stats_t* h_stats);
vmps_status_t vmps_sort_pairs_host(const void* h_keys, const uint32_t* h_vals, void* h_keys_out,
                                   uint32_t* h_vals_out, uint64_t n, vmps_key_t kt, int64_t scratch_elems,
                                   void* d_keys, uint32_t* d_vals, void* ws, size_t ws_bytes, void* stream,
                                   vmps_stats_t* h_stats);

/* The merge plan of Alg. 1 for keys[0,n) (keys are only read):
 * run_start[r] (ascending, run_start[0] = 0), run_kind[r] (VMPS_RUN_* bits),
 * merges[r-1] in Alg. 1's execution order.  cap_runs = capacity of
 * run_start/run_kind (merges needs cap_runs - 1).  *h_num_runs receives r
 * (synchronises); if r > cap_runs nothing is written and
 * VMPS_ERR_INVALID_ARG is returned. */
vmps_status_t vmps_merge_plan(const void* keys, uint64_t n, vmps_key_t kt, uint64_t* run_start,
                              uint8_t* run_kind, vmps_merge_rec_t* merges, uint64_t cap_runs,
                              uint64_t* h_num_runs, void* ws, size_t ws_bytes, void* stream);

/* ---- multi-GPU building blocks (BASELINE.json north_star) ----
 * A sharded sort runs on every rank: local vmps_sort_pairs, exact splitters
 * by a distributed binary search over the key order image using
 * vmps_count_rank, an NCCL all-to-all of the pieces (torch.distributed), and
 * vmps_merge_runs over the received pieces (ordered by source rank).
 *
 * vmps_count_rank: keys[0,n) sorted under the key order; probes[p] (device,
 * u64) are values of the order image (u32/u64 as is; f32 the image that
 * makes -0.0 < +0.0 and NaNs last and equal, as a u32 in the low bits).
 * Writes out_lt[p] = #{x : img(x) < probes[p]} and out_le[p] = #{x : img(x)
 * <= probes[p]} (device u64 arrays).  Stream-ordered, no synchronisation. */
vmps_status_t vmps_count_rank(const void* keys, uint64_t n, vmps_key_t kt, const uint64_t* probes,
                              uint32_t nprobe, uint64_t* out_lt, uint64_t* out_le, void* stream);

/* ---- distributed merge plan ----
 * The plan of the concatenation of g shards (rank q holds keys[off_q,
 * off_q + n_q) of the global array) is Alg. 1's plan of the whole array with
 * the global n (reading R15/C13).  Building blocks, one call per
 * rank, composed by paper_2605_27147_b200.dist.merge_plan_dist:
 *
 * vmps_shard_chain: the shard's transfer table of the run-detection chain
 * (ExtractRun, P:399 / P:756, with the global minrun): for every chain state
 * s at the shard start (START(o) = o, ASC(f) = minrun + f, DESC(f) = 2 minrun
 * + f, o, f < minrun; END = 255), d_table[s] = (state at the shard end << 32)
 * | runs started inside the shard.  n_end = the global n minus the shard's
 * offset (where the chain ends, relative to the shard start), or 0xFFFFFFFF
 * if that is >= 2^32 - 1.  d_prev: device pointer to the previous shard's last
 * key (NULL for shard 0); d_halo: the next n_halo <= 136 keys of the global
 * array after this shard (>= minrun + 2 of them unless the array ends
 * sooner), so runs crossing the shard end are classified exactly.  d_table:
 * device, 3 minrun u64.  n_local <= VMPS_MAX_N.
 *
 * vmps_shard_runs: with the chain state at the shard start (composition of the
 * previous shards' tables from START(0)), writes the shard's `count` run
 * starts (global positions offset + local, u64) and kinds (VMPS_RUN_* bits)
 * to device arrays.  count = d_table[entry_state] & 0xFFFFFFFF.
 *
 * Workspace for both: vmps_shard_workspace_bytes(n_local, kt, minrun).
 *
 * vmps_plan_from_runs: the merge plan (r - 1 records in Alg. 1's execution
 * order, as vmps_merge_plan) of an array of n keys whose r runs start at
 * d_run_start[0..r) (64-bit global positions, d_run_start[r] = n).  Workspace:
 * vmps_plan_workspace_bytes(r).  Synchronises `stream`. */
vmps_status_t vmps_shard_workspace_bytes(uint64_t n_local, vmps_key_t kt, uint32_t minrun, size_t* h_bytes);
vmps_status_t vmps_shard_chain(const void* keys, uint64_t n_local, vmps_key_t kt, uint32_t minrun, uint32_t n_end,
                               const void* d_prev, const void* d_halo, uint32_t n_halo, uint64_t* d_table,
                               void* ws, size_t ws_bytes, void* stream);
vmps_status_t vmps_shard_runs(const void* keys, uint64_t n_local, vmps_key_t kt, uint32_t minrun, uint32_t n_end,
                              const void* d_prev, const void* d_halo, uint32_t n_halo, uint32_t entry_state,
                              uint64_t count, uint64_t offset, uint64_t* d_run_start, uint8_t* d_run_kind, void* ws,
                              size_t ws_bytes, void* stream);
vmps_status_t vmps_plan_workspace_bytes(uint64_t r, size_t* h_bytes);
vmps_status_t vmps_plan_from_runs(const uint64_t* d_run_start, uint64_t r, uint64_t n, vmps_merge_rec_t* d_merges,
                                  void* ws, size_t ws_bytes, void* stream);

/* ---- native multi-GPU entry points; paper_2605_27147_b200/csrc/comm.cu ----
 * One process per GPU; NCCL (loaded with dlopen on first use) carries the
 * exchanges.  A communicator: rank 0 calls vmps_comm_unique_id and shares the
 * 128 bytes with the other ranks out of band (e.g. a torch.distributed
 * broadcast); every rank calls vmps_comm_init(&c, rank, world, id, device).
 * Errors of these calls: VMPS_ERR_NCCL / VMPS_ERR_CUDA with detail in
 * vmps_comm_last_error().
 *
 * vmps_sort_keys_dist / vmps_sort_pairs_dist: the globally stable sort of the
 * concatenation of the ranks' shards (rank order), in place: rank p ends with
 * the global output ranks [off_p, off_p + n_local_p), off_p = sum of the
 * earlier ranks' n_local, so each rank keeps its element count.  Steps: local
 * vmps_sort_*; exact splitters for the output ranks off_1..off_{g-1} by a
 * 16-ary search over the key order image (vmps_count_rank counts, summed by
 * ncclAllReduce; 8 rounds for u32/f32, 16 for u64); the tie group at each
 * splitter is split in rank order (lower ranks first: stability); grouped
 * ncclSend / ncclRecv of keys and payloads; vmps_merge_runs of the received
 * pieces in source-rank order (ties to the lower rank).  h_stats (optional)
 * reports the local sort.  Workspace: vmps_dist_workspace_bytes.  Synchronises
 * `stream` once per search round (each wait polls for NCCL errors and the
 * VMPS_COMM_TIMEOUT_S timeout).
 *
 * vmps_merge_plan_dist: Alg. 1's merge plan of the concatenated shards with
 * the global n (reading C13; as paper_2605_27147_b200.dist.merge_plan_dist):
 * each rank receives the runs starting in its shard (global u64 positions,
 * kinds) and the merges whose boundary j lies in its shard, in Alg. 1's order
 * (the `order` field is the global execution rank); cap_runs bounds both
 * outputs.  Workspace: vmps_merge_plan_dist_workspace_bytes(n_total, ...),
 * n_total = the sum of all shard sizes.  Synchronises `stream`. */
typedef struct vmps_comm_s* vmps_comm_t;
vmps_status_t vmps_comm_unique_id(void* h_id128);
vmps_status_t vmps_comm_init(vmps_comm_t* h_out, int rank, int world, const void* h_id128, int device);
vmps_status_t vmps_comm_destroy(vmps_comm_t c);
const char* vmps_comm_last_error(void);
vmps_status_t vmps_dist_workspace_bytes(uint64_t n_local, vmps_key_t kt, int has_vals, int world,
                                        int64_t scratch_elems, size_t* h_bytes);
vmps_status_t vmps_sort_keys_dist(vmps_comm_t c, void* keys, uint64_t n_local, vmps_key_t kt, int64_t scratch_elems,
                                  void* ws, size_t ws_bytes, void* stream, vmps_stats_t* h_stats);
vmps_status_t vmps_sort_pairs_dist(vmps_comm_t c, void* keys, uint32_t* vals, uint64_t n_local, vmps_key_t kt,
                                   int64_t scratch_elems, void* ws, size_t ws_bytes, void* stream,
                                   vmps_stats_t* h_stats);
vmps_status_t vmps_merge_plan_dist_workspace_bytes(uint64_t n_total, uint64_t n_local, vmps_key_t kt, int world,
                                                   size_t* h_bytes);
/* cap_runs that always suffices for vmps_merge_plan_dist on this shard:
 * n_local / minrun(n_total) + 2 (every run but the array's last has >= minrun
 * keys; merges with j in the shard are at most as many as its runs). */
vmps_status_t vmps_merge_plan_dist_capacity(uint64_t n_total, uint64_t n_local, uint64_t* h_cap);
vmps_status_t vmps_merge_plan_dist(vmps_comm_t c, const void* keys, uint64_t n_local, vmps_key_t kt,
                                   uint64_t* run_start, uint8_t* run_kind, vmps_merge_rec_t* merges,
                                   uint64_t cap_runs, uint64_t* h_num_runs_local, uint64_t* h_num_merges_local,
                                   void* ws, size_t ws_bytes, void* stream);

/* In-process virtual ranks (tests): vmps_local_group_create
 * makes a group of `world` ranks that are threads of this process (any
 * devices; all on one GPU is the intended use), vmps_comm_init_local gives
 * rank `rank` its communicator.  Every vmps_*_dist call then runs the same
 * protocol as over NCCL, with collectives made of host barriers, CUDA events
 * and device-to-device copies; each rank calls from its own thread with its
 * own stream and workspace.  A rank that does not reach a collective within
 * VMPS_COMM_TIMEOUT_S seconds (default 600) fails the group: every waiting
 * call returns VMPS_ERR_NCCL.  Destroy the communicators before the group.
 *
 * Failure detection (both transports): every host wait of the protocol polls
 * the stream, and for NCCL ncclCommGetAsyncError; an asynchronous NCCL error
 * or a wait longer than VMPS_COMM_TIMEOUT_S aborts the communicator and
 * returns VMPS_ERR_NCCL (detail in vmps_comm_last_error()). */
vmps_status_t vmps_local_group_create(int world, int device, void** h_group);
vmps_status_t vmps_local_group_destroy(void* group);
vmps_status_t vmps_comm_init_local(vmps_comm_t* h_out, int rank, void* group, int device);

/* vmps_dist_cuts: steps 2-3 of the distributed sort on already sorted shards
 * (used by the pull-merge protocol): every rank's shard size (h_sizes[g],
 * optional) and the exact cut table h_cut[q * (g + 1) + t] = elements of rank
 * q that go to ranks < t (global output ranks [off_t, off_t+1) go to rank t,
 * ties split in rank order).  h_rounds (optional): search rounds.  Workspace:
 * vmps_dist_cuts_workspace_bytes(world).  Synchronises `stream`. */
vmps_status_t vmps_dist_cuts_workspace_bytes(int world, size_t* h_bytes);
vmps_status_t vmps_dist_cuts(vmps_comm_t c, const void* keys, uint64_t n_local, vmps_key_t kt, uint64_t* h_cut,
                             uint64_t* h_sizes, uint32_t* h_rounds, void* ws, size_t ws_bytes, void* stream);

/* ---- host-side protocol arithmetic (no device work; the native protocol's
 * own steps, exported so other orchestrations and CPU tests use them) ----
 * vmps_splitter_probes: the probes of one 16-ary search round of the m
 * splitters over the key order image: for each t with lo[t] < hi[t], up to
 * 15 increasing probes in [lo[t], hi[t]) at lo + k (hi - lo) / 16; h_probe
 * (capacity 15 m) receives them, h_base[m + 1] the index of each splitter's
 * first probe, *h_nprobe the count (0 = every splitter found).
 * vmps_splitter_update: with h_le_sum[k] = #{keys of all ranks with image <=
 * probe k}, narrows [lo[t], hi[t]] to the least image v with #{<= v} >= R[t].
 * vmps_split_points: per-rank cut for output rank R from every rank's counts
 * of '< v*' (h_lt[g]) and '<= v*' (h_le[g]): all keys < v*, then the tie group
 * at v* in rank order (stability).
 * vmps_compose_tables: composition of g shards' run-detection transfer tables
 * (h_tables[q * ns + state], see vmps_shard_chain) from START(0): each shard's
 * entry state and runs started (empty shards: identity). */
vmps_status_t vmps_splitter_probes(uint32_t m, const uint64_t* h_lo, const uint64_t* h_hi, uint64_t* h_probe,
                                   uint32_t* h_base, uint32_t* h_nprobe);
vmps_status_t vmps_splitter_update(uint32_t m, uint64_t* h_lo, uint64_t* h_hi, const uint64_t* h_R,
                                   const uint64_t* h_probe, const uint32_t* h_base, const uint64_t* h_le_sum);
vmps_status_t vmps_split_points(uint32_t g, uint64_t R, const uint64_t* h_lt, const uint64_t* h_le, uint64_t* h_cut);
vmps_status_t vmps_compose_tables(uint32_t g, uint32_t ns, const uint64_t* h_tables, const uint64_t* h_sizes,
                                  uint32_t* h_entry, uint64_t* h_count);

/* ---- pull-merge (csrc/engine4.cuh k_pull_merge) ----
 * vmps_merge_pieces: the stable merge of g (1..8) sorted pieces that live at
 * arbitrary device addresses -- on a multi-GPU box the co-ranked pieces of
 * the other ranks' shards, mapped with vmps_ipc_open (CUDA IPC over NVLink)
 * -- written once into out_keys / out_vals [0, N), N = sum of h_counts.
 * Ties go to the lower piece index (the lower source rank).  h_keys /
 * h_vals / h_counts are host arrays of g entries; h_vals and out_vals may be
 * NULL (keys only).  Pieces are read by TMA bulk copies aligned down / up to
 * 16 bytes, so each piece must lie in an allocation that covers those bytes
 * (any cudaMalloc allocation does).  g <= 4: one pass of the 4-way engine;
 * g <= 8: two such passes into the two halves of the output, then one local
 * 2-way merge (vmps_merge_runs).  Workspace:
 * vmps_merge_pieces_workspace_bytes.
 *
 * vmps_ipc_handle: the CUDA IPC handle (64 bytes) of the allocation holding
 * d_ptr and d_ptr's offset in it; vmps_ipc_open maps a peer's handle and
 * returns base + offset; vmps_ipc_close unmaps (pass the same offset).
 * Errors: VMPS_ERR_CUDA with detail in vmps_comm_last_error(). */
vmps_status_t vmps_merge_pieces_workspace_bytes(uint64_t n_total, vmps_key_t kt, int has_vals, uint32_t g,
                                                size_t* h_bytes);
vmps_status_t vmps_merge_pieces(const void* const* h_keys, const uint32_t* const* h_vals, const uint64_t* h_counts,
                                uint32_t g, void* out_keys, uint32_t* out_vals, vmps_key_t kt, void* ws,
                                size_t ws_bytes, void* stream);
vmps_status_t vmps_ipc_handle(const void* d_ptr, void* h_handle64, uint64_t* h_offset);
vmps_status_t vmps_ipc_open(const void* h_handle64, uint64_t offset, void** h_ptr);
vmps_status_t vmps_ipc_close(void* d_ptr, uint64_t offset);

/* ---- large records (paper_2605_27147_b200/csrc/records.cu) ----
 * vmps_sort_records: n records of `words` u32 each (row-major, device),
 * ordered lexicographically with word 0 most significant (the paper's blob
 * types: arrays of 30 ints ordered lexicographically), sorted
 * stably.  The engine sorts (64-bit word-pair key, u32 index) pairs: by the
 * first word pair that is not equal in every record, and, only if two
 * records tie on it while a later pair varies, an LSD pass per varying word
 * pair from the last to that one; then one gather writes records_out (may be NULL; must not alias
 * records).  perm_out (may be NULL, u32[n]) receives the permutation: the
 * paper's `ptr` type (pointers sorted by their arrays).  n <= VMPS_MAX_N.
 * Workspace: vmps_sort_records_workspace_bytes.  May synchronise `stream`
 * (tie check).  Error detail: vmps_records_last_error(). */
vmps_status_t vmps_sort_records_workspace_bytes(uint64_t n, uint32_t words, size_t* h_bytes);
vmps_status_t vmps_sort_records(const uint32_t* records, uint32_t* records_out, uint32_t* perm_out, uint64_t n,
                                uint32_t words, void* ws, size_t ws_bytes, void* stream);
const char* vmps_records_last_error(void);

/* vmps_merge_runs: keys[0,n) (and vals, if non-NULL) consist of nruns adjacent
 * runs, each sorted, starting at h_run_start[0] = 0 < h_run_start[1] < ...
 * (host array).  Merges them in place into the stable sort of the array,
 * ties to the earlier run (Alg. 2 tie rule), along a balanced tree of
 * pairwise merges executed level by level on the level-merge engine.
 * Workspace: vmps_merge_runs_workspace_bytes.  Synchronises `stream` once
 * (to upload the small tree description). */
vmps_status_t vmps_merge_runs_workspace_bytes(uint64_t n, vmps_key_t kt, int has_vals,
                                              uint32_t nruns, size_t* h_bytes);
vmps_status_t vmps_merge_runs(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt,
                              const uint64_t* h_run_start, uint32_t nruns, void* ws,
                              size_t ws_bytes, void* stream);

/* vmps_merge_runs_bounded: as vmps_merge_runs (adjacent sorted runs starting
 * at h_run_start[0] = 0 < ... < n, host array; ties to the earlier run), with
 * the element scratch capped at scratch_elems like the bounded sort (block
 * table, level passes into freed blocks, final Copy); the plan is built from
 * the given runs (no run detection), so its metadata is O(nruns + n / P).
 * Workspace: vmps_merge_runs_bounded_workspace_bytes.  Synchronises `stream`
 * (the bounded mode's error check). */
vmps_status_t vmps_merge_runs_bounded_workspace_bytes(uint64_t n, vmps_key_t kt, int has_vals, uint32_t nruns,
                                                      int64_t scratch_elems, size_t* h_bytes);
vmps_status_t vmps_merge_runs_bounded(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt,
                                      const uint64_t* h_run_start, uint32_t nruns, int64_t scratch_elems, void* ws,
                                      size_t ws_bytes, void* stream);

/* Human-readable status; the last CUDA error detail of this thread. */
const char* vmps_status_string(vmps_status_t s);
const char* vmps_last_error(void);

/* Bench hooks (process-global, not thread safe).  With profiling on, each
 * sort records CUDA events on its stream around its phases; after the stream
 * is synchronised, vmps_profile_read fills h_ms[0..cap): [0] run detection +
 * plan, [1] leaf engine, [2] all level partitions, [3] all level merges,
 * [4] total; h_launches[0] = kernels launched by the last sort, h_launches[1]
 * = level-merge launches, h_bytes[0] = algorithmic bytes of the level merges
 * (2 w (M - fused M)).  Returns the number of values written. */
void vmps_profile_enable(int on);
int vmps_profile_read(double* h_ms, int cap, uint64_t* h_launches, uint64_t* h_bytes);

/* Test-only hooks (process-global, not thread safe).  minrun = 0 restores
 * the paper's rule; otherwise 1..64 forces minrun.  Z (fused-subtree limit),
 * T_out (merge tile) and P_blk (bounded block) = 0 restore defaults. */
void vmps_test_set_minrun(uint32_t minrun);
/* Test hook: merge schedule.  2 (default, also 0): two tree levels per HBM
 * pass -- only even-depth nodes are materialized and each merges up to four
 * runs (its grandchildren) in one pass, so every element is read and written
 * about half as often; 1: one level (one 2-way merge) per pass.  Same output. */
void vmps_test_set_mode(int levels_per_pass);
/* Test hook: leaf engine.  0 (default): block merge sort of each leaf batch
 * in shared memory (k_leaf_sort); 1: LSD radix sort (k_leaf_radix, slower at
 * 2^30 cfg5: 29 vs 18 ms).  Same output (a stable sort is unique). */
void vmps_test_set_leaf(int radix);
void vmps_test_set_tiles(uint32_t fuse_z, uint32_t merge_tile, uint32_t block_elems);
/* Test hook: chunk of the chunked scratch-bounded mode (used when n > 2 chunk;
 * 0 restores 2^24): each chunk is sorted by the bounded engine, then the
 * sorted chunks are merged along their Powersort tree, so the plan metadata
 * scales with the chunk instead of n.  Same output. */
void vmps_test_set_bd_chunk(uint32_t chunk);

#ifdef __cplusplus
}
#endif
#endif
