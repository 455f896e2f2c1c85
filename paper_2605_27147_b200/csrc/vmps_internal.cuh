// vmps_internal.cuh -- shared device/host definitions of libvmps (sm_100a).
// Product code: no dependency on oracle/ (see DESIGN.md "Independence").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vmps.h"

namespace vmps {

// ---------------------------------------------------------------------------
// Key order (reading R5).  Every compare maps a key to an unsigned
// image whose integer order is the sort order; keys are never rewritten.
// f32: NaN (any sign/payload) -> 0xFFFFFFFF (last, all equal); otherwise flip
// all bits of negatives and the sign bit of non-negatives (-0.0 < +0.0).
// ---------------------------------------------------------------------------
template <int KT>
struct KeyTraits;
template <>
struct KeyTraits<VMPS_KEY_U32> {
  using K = uint32_t;
  using O = uint32_t;
  __device__ __forceinline__ static O ord(K x) { return x; }
};
template <>
struct KeyTraits<VMPS_KEY_U64> {
  using K = uint64_t;
  using O = uint64_t;
  __device__ __forceinline__ static O ord(K x) { return x; }
};
template <>
struct KeyTraits<VMPS_KEY_F32> {
  using K = uint32_t;  // raw bits
  using O = uint32_t;
  __device__ __forceinline__ static O ord(K x) {
    if ((x & 0x7FFFFFFFu) > 0x7F800000u) return 0xFFFFFFFFu;
    return x ^ ((x & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u);
  }
};

// Run-chain states: START(o), ASC(f), DESC(f)
// for o, f in [0, minrun), plus END.
constexpr uint32_t ST_END = 255u;
constexpr int RT = 4096;             // run-detection tile (elements)
constexpr int RT_WORDS = RT / 32;    // bitmap words per tile
constexpr int CHAIN_G = 64;          // tables composed per group
constexpr int MAX_MINRUN = 64;
constexpr int MAX_NS = 3 * MAX_MINRUN;

// Plan / schedule defaults
#ifndef VMPS_FUSE_Z
#define VMPS_FUSE_Z 2048
#endif
constexpr uint32_t DEFAULT_FUSE_Z = VMPS_FUSE_Z;   // fused-subtree limit Z (elements)
constexpr uint32_t MAX_FUSE_Z = VMPS_FUSE_Z;
constexpr uint32_t MERGE_BLOCK = 512;       // threads per merge CTA
constexpr uint32_t MERGE_K = 8;             // outputs per thread
constexpr uint32_t DEFAULT_TOUT = MERGE_BLOCK * MERGE_K;  // merge tile (outputs)

// Device-side scalars (one small array in the workspace).
enum Scalar : int {
  SC_RUNS = 0,        // r
  SC_UNITS,           // number of fused units
  SC_LONG,            // number of long leaves
  SC_LONG_CHUNKS,     // chunks over long leaves
  SC_NONFUSED,        // number of non-fused nodes
  SC_MAXPOW,          // max node power
  SC_REVERSED,        // reversed elements
  SC_EXTENDED,        // extended runs
  SC_LEVEL_TILES,     // scratch for per-level tile count
  SC_ERROR,           // internal consistency error flag
  SC_NBATCH,          // leaf batches
  SC_LEAFQ,           // leaf work queues (2 slots: one per CTA size class)
  SC_LEAFQ1,
  SC_COUNT = 16
};
constexpr int LEVEL_SLOTS = 72;  // powers 0..70

// Device arrays carved from the caller's workspace.
struct Work {
  uint32_t n, minrun, ns, ntiles;
  uint32_t rmax;       // capacity for runs (+2 slack)
  uint32_t fuse_z, tout;
  uint32_t bcap;       // leaf batches (upper bound)
  int kt, has_vals;
  // element scratch (buffer 1 of the ping-pong pair)
  void* k1;
  uint32_t* v1;
  // run detection
  uint32_t* bits;      // (n/32 + 2) words, bit p = key[p] < key[p-1]
  uint32_t* tile_tab;  // ntiles * ns, (state << 24) | count
  uint64_t* chain_tab[4];  // composed levels
  uint32_t chain_m[5];     // table counts per level (0 = tiles)
  int chain_levels;        // number of composed levels
  uint64_t* chain_entry[5];// entry (state << 32 | count) per table per level
  uint32_t* run_start;     // rmax + 1
  uint8_t* run_kind;       // rmax
  uint32_t* scalars;       // SC_COUNT
  // plan (boundary t in [1, r-1]; arrays sized rmax)
  uint8_t* power;
  uint32_t* seg_l;    // first run of node t's segment
  uint32_t* seg_r;    // one past the last run
  uint32_t* parent;   // boundary index, 0 = root
  uint32_t* anc[2];   // pointer jumping
  uint32_t* dep[2];   // depth (low 16 bits) | left-ancestor count (high 16)
  // classification
  uint32_t* unit_flag;   // per run: 1 = unit start
  uint32_t* long_flag;   // per run: 1 = long leaf
  uint32_t* unit_end;    // per run (unit starts): end position
  uint8_t* unit_par;     // per run (unit starts): output buffer parity
  uint8_t* long_par;     // per run (long leaves): parity | desc << 1
  uint32_t* long_chunks; // per long leaf: chunks of work
  uint32_t* long_off;    // exclusive scan of long_chunks
  uint32_t* unit_idx;    // scan of unit_flag
  uint32_t* long_idx;    // scan of long_flag
  uint32_t* units;       // [3 * rmax]: start, end, parity (compacted)
  uint32_t* batch_first; // first unit of each leaf batch (n / Z + 2)
  uint32_t* longs;       // [4 * rmax]: start, end, parity|desc<<1, chunk offset
  uint32_t* level_cnt;   // LEVEL_SLOTS
  uint32_t* level_start; // LEVEL_SLOTS + 1 (node offsets)
  uint32_t* level_fill;  // LEVEL_SLOTS
  uint32_t* level_tile;  // LEVEL_SLOTS + 1 (tile offsets)
  uint32_t* lnodes;      // bucketed non-fused nodes
  uint32_t* ltiles_cnt;  // tiles per bucketed node
  uint32_t* ltiles;      // tile offset per bucketed node (exclusive scan)
  void* desc;            // TileDesc per tile of one level
  uint32_t part_cap;
  uint32_t* scan_tmp;    // block sums for scans
  uint64_t* gpos;        // given-runs mode: global run starts (powers with the global n)
  unsigned long long* counters;  // [0] M, [1] fused M
  // two-level fused merges (engine4.cuh)
  int fuse2;
  uint32_t *lchild, *rchild;
  void *nr4, *tiles4;
  uint32_t n4cap;
  // scratch-bounded mode (bounded.cuh); element scratch = F blocks of P
  int bounded;
  uint32_t P, F, NB;
  uint32_t *Tin, *Tout, *inv, *pool, *remain, *dirty, *didx, *dlist, *first_tile;
  uint32_t *bflag, *bpos, *blnodes, *bcnt, *btoff, *bm, *bD;
  uint32_t *lvl_hist, *lvl_hscan;  // level schedule: per-tile power histograms and their scan
  void* bdesc;
  uint32_t bdesc_cap;
  void* bstate;
  uint32_t* cplists;      // final Copy: two list sets (bounded.cuh BD_CP_LIST words each)
  // dyadic-cell mode: the block table (and element scratch) of the whole
  // array lives outside this sort (api.cu BdCtx); positions here are
  // relative to gt_base
  const void* gt_ctx;
  uint64_t gt_base;
  size_t scratch_bytes;
  size_t used_bytes;
};

}  // namespace vmps
