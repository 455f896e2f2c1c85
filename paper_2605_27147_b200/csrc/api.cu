// api.cu -- C ABI (include/vmps.h) and stream-ordered orchestration of the
// hot path: run detection -> powers / merge tree / schedule -> leaf engine ->
// one partition + one merge launch per tree level.  No host synchronisation
// happens between launches; only h_stats / h_num_runs read results back.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges per phase (no link dependency)

#include "bounded.cuh"
#include "engine.cuh"
#include "engine4.cuh"
#include "leaf_radix.cuh"
#include "plan.cuh"
#include "runs.cuh"
#include "vmps_internal.cuh"

namespace vmps {

static uint32_t g_minrun_override = 0;
static uint32_t g_fuse_z = 0;
static uint32_t g_tout = 0;
static uint32_t g_blk = 0;
static int g_fuse2 = 1;  // two tree levels per merge pass (default; vmps_test_set_mode(1) = one)
static int g_leaf_radix = 0;  // test hook vmps_test_set_leaf  // two-level fused merges (opt-in, test hook vmps_test_set_mode)
static thread_local std::string g_err;

// ---- bench profiling (process-global) ----
static bool g_prof = false;
static cudaEvent_t g_ev[256];
static bool g_ev_init = false;
static int g_ev_n = 0;
static uint64_t g_nl = 0;         // kernels launched by the current sort
static uint64_t g_nl_merge = 0;   // level-merge launches
static int g_prof_lvl[128][2];    // (start, end) event index per merge launch
static int g_prof_part[128][2];   // per partition launch
static int g_prof_nm = 0, g_prof_np = 0;
static int g_prof_mark[4] = {-1, -1, -1, -1};  // begin, after plan, after leaf, end
static unsigned long long* g_prof_host = nullptr;  // pinned copy of counters
static int g_prof_wbytes = 0;

// NVTX ranges around the host-side enqueue of each phase (visible to
// Nsight tools; `ncu --nvtx --nvtx-include "vmps_sort/vmps_merge/"` selects a phase).
struct NvtxRange {
  bool on = true;
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  void end() { if (on) { nvtxRangePop(); on = false; } }
  ~NvtxRange() { end(); }
};

static int prof_event(cudaStream_t s) {
  if (!g_prof || g_ev_n >= 256) return -1;
  if (!g_ev_init) {
    for (int i = 0; i < 256; ++i) cudaEventCreate(&g_ev[i]);
    cudaHostAlloc((void**)&g_prof_host, 64, cudaHostAllocDefault);
    g_ev_init = true;
  }
  cudaEventRecord(g_ev[g_ev_n], s);
  return g_ev_n++;
}
static void prof_reset() {
  g_ev_n = 0;
  g_nl = 0;
  g_nl_merge = 0;
  g_prof_nm = g_prof_np = 0;
  for (int i = 0; i < 4; ++i) g_prof_mark[i] = -1;
}

static uint32_t minrun_rule(uint64_t n) {
  uint64_t l = n;
  while (l >= 64) l = (l + 1) / 2;
  return (uint32_t)l;
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }
#ifndef VMPS_LEAF_ZB_SMALL
#define VMPS_LEAF_ZB_SMALL 1
#endif
// Leaf batch window Zb: a batch (touching units starting in one window) spans
// < Zb + Z positions.  VMPS_LEAF_ZB_SMALL: windows sized for the half-size CTA
// (every batch fits it; cfg5 leaf 12.88 -> 12.64 ms), except in the bounded
// mode, whose metadata (n / Zb batch slots) must stay small.
static uint32_t leaf_zb(uint32_t fuse_z, bool bounded) {
  const bool small = VMPS_LEAF_ZB_SMALL && !bounded && (uint32_t)LEAF_SMALL_CAP > fuse_z;
  return (small ? (uint32_t)LEAF_SMALL_CAP : (uint32_t)LEAF_CAP) - fuse_z + 1;
}

#ifndef VMPS_DESC4_WARP_MAX_BIG
#define VMPS_DESC4_WARP_MAX_BIG 4096u  // warp-per-tile partition below this many tiles, arrays > 512 MB of keys
#endif
#ifndef VMPS_SCAN1
#define VMPS_SCAN1 1
#endif
static size_t scan_tmp_words(size_t len) {
  size_t nb = (len + SCAN_TILE - 1) / SCAN_TILE;
  if (nb <= 1) return 2;
  return 2 * nb + scan_tmp_words(nb);
}

struct Cfg {
  uint64_t n;
  int kt;
  int hv;         // 1 with payload, 0 keys only, -1 plan only
  uint32_t minrun, fuse_z, tout;
  int64_t scratch;  // VMPS_SCRATCH_UNBOUNDED or the element cap
  int fuse2;
  uint32_t P, F;    // bounded mode: block size, scratch blocks
  uint32_t given_runs;  // > 0: the runs are given (no run detection; per-run arrays sized by it)
  uint32_t gt_nb = 0;   // > 0: the block table is external (the whole array's, gt_nb blocks)
};

static Cfg make_cfg(uint64_t n, int kt, int hv, int64_t scratch = VMPS_SCRATCH_UNBOUNDED) {
  Cfg c;
  c.n = n;
  c.kt = kt;
  c.hv = hv;
  c.minrun = g_minrun_override ? g_minrun_override : minrun_rule(n);
  c.fuse_z = g_fuse_z ? g_fuse_z : DEFAULT_FUSE_Z;
  c.tout = g_tout ? g_tout : DEFAULT_TOUT;
  c.scratch = scratch;
  c.fuse2 = (scratch < 0 && hv >= 0) ? g_fuse2 : 0;
  c.P = c.F = 0;
  c.given_runs = 0;
  if (scratch >= 0 && hv >= 0) {
    // block size: a power of two <= min(Z, T_out) (nodes are then longer than
    // a block, so a block meets at most 3 tile pieces), test hook override
    // default: the largest power of two <= S / 16 (>= 16 scratch blocks)
    uint32_t P = g_blk ? g_blk : (uint32_t)std::max<int64_t>(16, std::min<int64_t>(scratch / 16, DEFAULT_TOUT));
    P = std::min(P, std::min(c.fuse_z, (uint32_t)DEFAULT_TOUT));
    P = std::min(P, BD_THREADS * MERGE_K);  // a level-pass CTA holds one block's outputs in registers
    uint32_t p2 = 16;
    while (p2 * 2 <= P) p2 *= 2;
    c.P = p2;
    c.F = (uint32_t)std::min<int64_t>(scratch / (int64_t)c.P, (int64_t)(n / c.P + 8));
    c.tout = c.P;  // tiles = blocks
  }
  return c;
}
constexpr uint32_t BD_MIN_BLOCKS = 6;

static size_t key_bytes(int kt) { return kt == VMPS_KEY_U64 ? 8 : 4; }

// Carve the workspace; with base == nullptr only the size is computed.
static size_t carve(const Cfg& c, Work* w, char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> void* {
    void* p = base ? (void*)(base + off) : nullptr;
    off += align_up(bytes);
    return p;
  };
  const uint64_t n = c.n;
  Work t;
  memset(&t, 0, sizeof(t));
  t.n = (uint32_t)n;
  t.minrun = c.minrun;
  t.ns = 3 * c.minrun;
  t.ntiles = c.given_runs ? 0u : (uint32_t)((n + RT - 1) / RT);
  t.rmax = c.given_runs ? c.given_runs + 2u : (uint32_t)(n / std::max<uint32_t>(c.minrun, 1) + 2);
  t.fuse_z = c.fuse_z;
  t.tout = c.tout;
  t.kt = c.kt;
  t.has_vals = c.hv;
  const size_t R = (size_t)t.rmax + 2;
  t.bounded = c.scratch >= 0 && c.hv >= 0;
  if (c.hv >= 0 && !c.gt_nb) {
    const size_t se = t.bounded ? (size_t)c.F * c.P : (size_t)n;  // element scratch
    t.k1 = take(se * key_bytes(c.kt));
    t.v1 = c.hv ? (uint32_t*)take(se * 4) : nullptr;
    t.scratch_bytes = se * (key_bytes(c.kt) + (c.hv ? 4 : 0));
  }
  t.bits = (uint32_t*)take(((size_t)t.ntiles * RT_WORDS + RT_WORDS + 8) * 4);
  t.tile_tab = (uint32_t*)take((size_t)t.ntiles * t.ns * 4);
  uint32_t m = t.ntiles;
  t.chain_m[0] = m;
  t.chain_levels = 0;
  while (m > (uint32_t)CHAIN_G) {
    m = (m + CHAIN_G - 1) / CHAIN_G;
    t.chain_tab[t.chain_levels] = (uint64_t*)take((size_t)m * t.ns * 8);
    t.chain_levels++;
    t.chain_m[t.chain_levels] = m;
  }
  for (int l = 0; l <= t.chain_levels; ++l) t.chain_entry[l] = (uint64_t*)take((size_t)t.chain_m[l] * 8);
  t.run_start = (uint32_t*)take(R * 4);
  t.run_kind = (uint8_t*)take(R);
  t.gpos = c.given_runs ? (uint64_t*)take(R * 8) : nullptr;
  t.scalars = (uint32_t*)take(SC_COUNT * 4 + 64);
  t.power = (uint8_t*)take(R);
  t.seg_l = (uint32_t*)take(R * 4);
  t.seg_r = (uint32_t*)take(R * 4);
  t.parent = (uint32_t*)take(R * 4);
  t.anc[0] = (uint32_t*)take(R * 4);
  t.anc[1] = (uint32_t*)take(R * 4);
  t.dep[0] = (uint32_t*)take(R * 4);
  t.dep[1] = (uint32_t*)take(R * 4);
  if (c.hv >= 0) {
    t.unit_flag = (uint32_t*)take(R * 4);
    t.long_flag = (uint32_t*)take(R * 4);
    t.unit_end = (uint32_t*)take(R * 4);
    t.unit_par = (uint8_t*)take(R);
    t.long_par = (uint8_t*)take(R);
    t.unit_idx = (uint32_t*)take(R * 4);
    t.long_idx = (uint32_t*)take(R * 4);
    t.units = (uint32_t*)take(R * 3 * 4);
    t.bcap = (uint32_t)(n / leaf_zb(c.fuse_z, c.scratch >= 0) + n / c.fuse_z + 2);
    t.batch_first = (uint32_t*)take(((size_t)t.bcap + 2) * 4);
    t.longs = (uint32_t*)take(R * 4 * 4);
    t.long_chunks = (uint32_t*)take(R * 4);
    t.long_off = (uint32_t*)take(R * 4);
    t.level_cnt = (uint32_t*)take((LEVEL_SLOTS + 1) * 4);
    t.level_start = (uint32_t*)take((LEVEL_SLOTS + 1) * 4);
    t.level_fill = (uint32_t*)take((LEVEL_SLOTS + 1) * 4);
    t.level_tile = (uint32_t*)take((LEVEL_SLOTS + 1) * 4);
    // level schedule of the unbounded engines (the bounded mode builds its
    // own per-level lists)
    t.part_cap = (uint32_t)(n / c.tout + 2 * (n / c.fuse_z) + 8);
    if (!t.bounded) {
      t.lnodes = (uint32_t*)take(R * 4);
      t.ltiles = (uint32_t*)take(R * 4);
      t.ltiles_cnt = (uint32_t*)take(R * 4);
      // tiles of one level: its nodes are disjoint and larger than Z, and a node
      // [i,k) spans ceil(k/T) - floor(i/T) <= (k-i)/T + 2 aligned tiles
      t.desc = take((size_t)t.part_cap * sizeof(TileDesc));
    }
    // the bounded mode also scans its dirty-block flags (NB + 1 entries),
    // which exceed R when the block is smaller than minrun
    const size_t nbs = c.gt_nb ? (size_t)c.gt_nb : (size_t)((n + c.P - 1) / c.P);
    const size_t nlt = ((size_t)t.rmax + BD_LVL_TILE) / BD_LVL_TILE;  // level-schedule tiles over [0, rmax]
    const size_t scan_len = t.bounded ? std::max<size_t>(std::max<size_t>(R, nbs + 1), BD_LVL_BINS * nlt + 1) : R;
    t.scan_tmp = (uint32_t*)take(scan_tmp_words(scan_len) * 4 + 64);
  }
  t.counters = (unsigned long long*)take(8 * 8);
  t.fuse2 = c.fuse2;
  if (t.fuse2) {
    t.lchild = (uint32_t*)take(R * 4);
    t.rchild = (uint32_t*)take(R * 4);
    t.n4cap = (uint32_t)(n / c.fuse_z + 4);
    t.nr4 = take((size_t)t.n4cap * sizeof(NodeRuns));
    t.tiles4 = take((size_t)t.part_cap * sizeof(TileDesc4));
  }
  if (t.bounded) {
    t.P = c.P;
    t.F = c.F;
    t.NB = (uint32_t)((n + c.P - 1) / c.P);
    // per-level lists of the rounds reuse arrays that are dead by then: the
    // pointer-jumping temporaries (anc, dep[1]) and the long-leaf compaction
    // flags (long_flag, long_idx), all R entries of 4 bytes
    t.bflag = t.anc[0];
    t.bpos = t.anc[1];
    t.blnodes = t.dep[1];
    t.bcnt = t.long_flag;
    t.btoff = t.long_idx;
    t.bm = (uint32_t*)take(64);
    t.bD = (uint32_t*)take(64);
    const size_t nlt = ((size_t)t.rmax + BD_LVL_TILE) / BD_LVL_TILE;
    t.lvl_hist = (uint32_t*)take((BD_LVL_BINS * nlt + 1) * 4);
    t.lvl_hscan = (uint32_t*)take((BD_LVL_BINS * nlt + 1) * 4);
  }
  if (t.bounded && !c.gt_nb) {
    const size_t NBp = (size_t)t.NB + 8, NP = (size_t)t.NB + c.F + 8;
    t.Tin = (uint32_t*)take(NBp * 4);
    t.Tout = (uint32_t*)take(NBp * 4);
    t.inv = (uint32_t*)take(NP * 4);
    t.pool = (uint32_t*)take(NP * 4);
    t.remain = (uint32_t*)take(NBp * 4);
    t.dirty = (uint32_t*)take(NBp * 4);
    t.didx = (uint32_t*)take(NBp * 4);
    t.dlist = (uint32_t*)take(NBp * 4);
    t.first_tile = (uint32_t*)take(NBp * 4);
    // tiles of one level: one per output block plus gap tiles at node ends
    t.bdesc_cap = (uint32_t)(n / c.P + 4 * std::min<uint64_t>(n / c.fuse_z, (uint64_t)t.rmax) + 16);
    t.bdesc = take((size_t)t.bdesc_cap * sizeof(BdTile));
    t.bstate = take(sizeof(BdState));
    t.cplists = (uint32_t*)take((size_t)2 * BD_CP_LIST * 4);
  }
  t.used_bytes = off;
  if (w) *w = t;
  return off;
}

// Internal non-blocking stream (per device) used to capture CUDA graphs.
constexpr int MAX_DEV = 16;
// Per-device caches (function attributes are set per device): the current
// device, clamped into the cache tables.
static int dev_slot() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0) d = 0;
  return d % MAX_DEV;
}
static int g_nsm = 0;
static int nsm() {
  if (!g_nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, dev);
    if (g_nsm <= 0) g_nsm = 148;
  }
  return g_nsm;
}

static unsigned grid_for(size_t items, unsigned threads = 256) {
  size_t g = (items + threads - 1) / threads;
  size_t cap = (size_t)nsm() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// Exclusive scan of len u32 (out[len-1] meaningful); tmp from scan_tmp_words.
static void scan_u32(const uint32_t* in, uint32_t* out, uint32_t len, uint32_t* tmp, cudaStream_t s) {
  if (VMPS_SCAN1 && len > 0) {  // single pass; the tile status words fit in tmp (len / 2048 + 2 words)
    const uint32_t nt = (len + SCAN1_TILE - 1) / SCAN1_TILE;
    unsigned long long* st = reinterpret_cast<unsigned long long*>(((uintptr_t)tmp + 7) & ~(uintptr_t)7);
    cudaMemsetAsync(st, 0, (size_t)nt * 8, s);
    k_scan1<<<nt, SCAN1_THREADS, 0, s>>>(in, out, len, st);
    ++g_nl;
    return;
  }
  uint32_t nb = (len + SCAN_TILE - 1) / SCAN_TILE;
  k_scan_tiles<<<nb, SCAN_THREADS, 0, s>>>(in, out, len, tmp);
  ++g_nl;
  if (nb > 1) {
    scan_u32(tmp, tmp + nb, nb, tmp + 2 * nb, s);
    k_scan_add<<<nb, SCAN_THREADS, 0, s>>>(out, len, tmp + nb);
    ++g_nl;
  }
}

#define VMPS_CK(call)                                                      \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) {                                               \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);         \
      return VMPS_ERR_CUDA;                                                \
    }                                                                      \
  } while (0)

static vmps_status_t launch_check() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string("kernel launch: ") + cudaGetErrorString(e);
    return VMPS_ERR_CUDA;
  }
  return VMPS_OK;
}

static bool g_chain_attrs[MAX_DEV] = {};
static vmps_status_t chain_attrs() {
  const int ds = dev_slot();
  if (g_chain_attrs[ds]) return VMPS_OK;
  const int sm = CHAIN_G * MAX_NS * 8;
  VMPS_CK(cudaFuncSetAttribute(k_chain_compose<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  VMPS_CK(cudaFuncSetAttribute(k_chain_compose<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  VMPS_CK(cudaFuncSetAttribute(k_chain_expand<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  VMPS_CK(cudaFuncSetAttribute(k_chain_expand<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  g_chain_attrs[ds] = true;
  return VMPS_OK;
}

// Launch helper: counts kernels for the bench's gpu_launches.
static int g_debug_sync = -1;  // VMPS_DEBUG_SYNC=1: synchronise + check after every launch
static bool debug_sync() {
  if (g_debug_sync < 0) {
    const char* e = getenv("VMPS_DEBUG_SYNC");
    g_debug_sync = (e && e[0] == '1') ? 1 : 0;
  }
  return g_debug_sync == 1;
}

// VMPS_BD_TRACE=1: host wall time per phase of the scratch-bounded mode
// (stream synchronised at each phase edge), printed to stderr per sort.
struct BdTrace {
  double t[12];
  long n[12];
};
static thread_local BdTrace g_bdt;
static int g_bd_trace = -1;
static bool bd_trace() {
  if (g_bd_trace < 0) {
    const char* e = getenv("VMPS_BD_TRACE");
    g_bd_trace = (e && e[0] == '1') ? 1 : 0;
  }
  return g_bd_trace == 1;
}
static double bd_now(cudaStream_t s) {
  if (!bd_trace()) return 0.0;
  cudaStreamSynchronize(s);
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static void bd_add(int slot, double t0, cudaStream_t s) {
  if (!bd_trace()) return;
  g_bdt.t[slot] += bd_now(s) - t0;
  g_bdt.n[slot]++;
}

#define LAUNCH(kern, grid, block, smem, stream, ...)                              \
  do {                                                                             \
    kern<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                      \
    ++g_nl;                                                                        \
    if (debug_sync()) {                                                            \
      cudaError_t e_ = cudaStreamSynchronize(stream);                              \
      if (e_ == cudaSuccess) e_ = cudaGetLastError();                              \
      if (e_ != cudaSuccess) {                                                     \
        g_err = std::string(#kern) + ": " + cudaGetErrorString(e_);               \
        fprintf(stderr, "vmps debug: %s\n", g_err.c_str());                      \
        return VMPS_ERR_CUDA;                                                      \
      }                                                                            \
    }                                                                              \
  } while (0)

// Run detection + plan front half (shared by sort and merge_plan).
template <int KT>
static vmps_status_t front_half(const Work& w, const void* keys, cudaStream_t s) {
  using K = typename KeyTraits<KT>::K;
  vmps_status_t arc = chain_attrs();
  if (arc != VMPS_OK) return arc;
  VMPS_CK(cudaMemsetAsync(w.scalars, 0, SC_COUNT * 4, s));
  VMPS_CK(cudaMemsetAsync(w.counters, 0, 8 * 8, s));
  LAUNCH(k_runs_tables<KT>, w.ntiles, 128, 0, s, (const K*)keys, w.n, w.minrun, w.ns, w.bits, w.tile_tab, w.n,
         (const K*)nullptr, (const K*)nullptr, 0u);
  // compose the chain of tile tables (level 0 = u32 tile tables, above = u64)
  const size_t sm32 = (size_t)CHAIN_G * w.ns * 4, sm64 = (size_t)CHAIN_G * w.ns * 8;
  for (int l = 0; l < w.chain_levels; ++l) {
    if (l == 0)
      LAUNCH(k_chain_compose<uint32_t>, w.chain_m[1], 256, sm32, s, w.tile_tab, w.chain_m[0], w.ns, w.chain_tab[0]);
    else
      LAUNCH(k_chain_compose<uint64_t>, w.chain_m[l + 1], 256, sm64, s, w.chain_tab[l - 1], w.chain_m[l], w.ns,
             w.chain_tab[l]);
  }
  const int top = w.chain_levels;
  if (top == 0)
    LAUNCH(k_chain_top<uint32_t>, 1, 32, 0, s, w.tile_tab, w.chain_m[0], w.ns, w.chain_entry[0], 0u);
  else
    LAUNCH(k_chain_top<uint64_t>, 1, 32, 0, s, w.chain_tab[top - 1], w.chain_m[top], w.ns, w.chain_entry[top], 0u);
  for (int l = top - 1; l >= 0; --l) {
    if (l == 0)
      LAUNCH(k_chain_expand<uint32_t>, w.chain_m[1], 256, sm32, s, w.tile_tab, w.chain_m[0], w.ns,
             w.chain_entry[1], w.chain_entry[0]);
    else
      LAUNCH(k_chain_expand<uint64_t>, w.chain_m[l + 1], 256, sm64, s, w.chain_tab[l - 1], w.chain_m[l], w.ns,
             w.chain_entry[l + 1], w.chain_entry[l]);
  }
  LAUNCH(k_runs_emit, w.ntiles, 128, 0, s, w.bits, w.n, w.minrun, w.chain_entry[0], w.run_start, w.run_kind,
         w.scalars, w.n, 0u);
  const unsigned g = grid_for(w.rmax);
  LAUNCH(k_powers_seg<uint32_t>, g, 256, 0, s, w.run_start, (uint64_t)w.n, w.scalars, w.power, w.seg_l, w.seg_r);
  LAUNCH(k_parent_init, g, 256, 0, s, w.scalars, w.power, w.seg_l, w.seg_r, w.parent, w.anc[0], w.dep[0]);
  // depth <= max power <= 34 < 64: six rounds of pointer jumping (result in dep[0])
  for (int rnd = 0; rnd < 6; ++rnd) {
    int a = rnd & 1;
    LAUNCH(k_jump, g, 256, 0, s, w.scalars, w.anc[a], w.dep[a], w.anc[a ^ 1], w.dep[a ^ 1]);
  }
  return launch_check();
}


// Given runs (the dyadic-cell scratch-bounded mode and the bounded merge of
// given runs): r runs at positions rel[0..r) of the sub-array (rel[r] = its
// length), their kinds (NULL: all ascending), and optionally their global
// positions gpos[0..r] in an array of n_glob elements -- then the node powers
// are the whole array's (P:445-446 with the global n), so the sub-array's
// tree is exactly the whole plan's subtree over these runs.
// The power of the boundary between [i, j) and [j, k) in an array of n
// (P:445-446): one plus the common leading bits of the two scaled midpoints.
static uint32_t host_power(uint64_t n, uint64_t i, uint64_t j, uint64_t k) {
  const unsigned __int128 N2 = (unsigned __int128)2 * n;
  unsigned __int128 A = (unsigned __int128)(i + j), B = (unsigned __int128)(j + k);
  uint32_t p = 0;
  for (;;) {
    ++p;
    A <<= 1;
    B <<= 1;
    const bool ba = A >= N2, bb = B >= N2;
    if (ba != bb) return p;
    if (ba) { A -= N2; B -= N2; }
  }
}

struct GivenRuns {
  const uint32_t* rel;
  const uint8_t* kinds;
  const uint64_t* gpos;
  uint64_t n_glob;
  uint32_t r;
  int p_min = 0;  // > 0: every boundary's power is >= p_min (a dyadic cell's runs), not recomputed
  // device-resident runs (dyadic-cell mode): global starts ring[(first + i) % cap]
  // and kinds, relative to `base`, the last ending at `end` (rel/kinds/gpos unused)
  const uint64_t* d_ring = nullptr;
  const uint8_t* d_ring_kind = nullptr;
  uint64_t ring_cap = 0, ring_first = 0, base = 0, end = 0;
  bool global() const { return gpos || d_ring; }
};

// Given runs from the device ring of the dyadic-cell mode.
__global__ void k_given_from_ring(uint32_t* __restrict__ rs, uint8_t* __restrict__ kind, uint64_t* __restrict__ gpos,
                                  uint32_t* __restrict__ scalars, const uint64_t* __restrict__ ring,
                                  const uint8_t* __restrict__ ring_kind, uint64_t cap, uint64_t first, uint32_t r,
                                  uint64_t base, uint64_t end) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= r; i += gridDim.x * blockDim.x) {
    const uint64_t g = i < r ? ring[(first + i) % cap] : end;
    rs[i] = (uint32_t)(g - base);
    gpos[i] = g;
    if (i < r) kind[i] = ring_kind[(first + i) % cap];
    if (i == 0) scalars[SC_RUNS] = r;
  }
}

static vmps_status_t front_half_given(const Work& w, const GivenRuns& G, cudaStream_t s) {
  const uint32_t r = G.r;
  VMPS_CK(cudaMemsetAsync(w.scalars, 0, SC_COUNT * 4, s));
  VMPS_CK(cudaMemsetAsync(w.counters, 0, 8 * 8, s));
  const unsigned g = grid_for(w.rmax);
  if (G.d_ring) {
    LAUNCH(k_given_from_ring, g, 256, 0, s, w.run_start, w.run_kind, w.gpos, w.scalars, G.d_ring, G.d_ring_kind,
           G.ring_cap, G.ring_first, r, G.base, G.end);
    LAUNCH(k_powers_seg<uint64_t>, g, 256, 0, s, w.gpos, G.n_glob, w.scalars, w.power, w.seg_l, w.seg_r);
    LAUNCH(k_parent_init, g, 256, 0, s, w.scalars, w.power, w.seg_l, w.seg_r, w.parent, w.anc[0], w.dep[0]);
    for (int rnd = 0; rnd < 6; ++rnd) {
      int a = rnd & 1;
      LAUNCH(k_jump, g, 256, 0, s, w.scalars, w.anc[a], w.dep[a], w.anc[a ^ 1], w.dep[a ^ 1]);
    }
    return launch_check();
  }
  VMPS_CK(cudaMemcpyAsync(w.run_start, G.rel, (size_t)(r + 1) * 4, cudaMemcpyHostToDevice, s));
  if (G.kinds) VMPS_CK(cudaMemcpyAsync(w.run_kind, G.kinds, r, cudaMemcpyHostToDevice, s));
  else VMPS_CK(cudaMemsetAsync(w.run_kind, 0, r, s));
  VMPS_CK(cudaMemcpyAsync(w.scalars + SC_RUNS, &r, 4, cudaMemcpyHostToDevice, s));
  if (G.gpos) {
    VMPS_CK(cudaMemcpyAsync(w.gpos, G.gpos, (size_t)(r + 1) * 8, cudaMemcpyHostToDevice, s));
    LAUNCH(k_powers_seg<uint64_t>, g, 256, 0, s, w.gpos, G.n_glob, w.scalars, w.power, w.seg_l, w.seg_r);
  } else {
    LAUNCH(k_powers_seg<uint32_t>, g, 256, 0, s, w.run_start, (uint64_t)w.n, w.scalars, w.power, w.seg_l, w.seg_r);
  }
  LAUNCH(k_parent_init, g, 256, 0, s, w.scalars, w.power, w.seg_l, w.seg_r, w.parent, w.anc[0], w.dep[0]);
  for (int rnd = 0; rnd < 6; ++rnd) {
    int a = rnd & 1;
    LAUNCH(k_jump, g, 256, 0, s, w.scalars, w.anc[a], w.dep[a], w.anc[a ^ 1], w.dep[a ^ 1]);
  }
  VMPS_CK(cudaStreamSynchronize(s));  // the host run lists are the caller's
  return launch_check();
}

// ---- scratch-bounded mode: level passes and the final Copy (bounded.cuh) ----
// The block table of one bounded sort: its own (one-piece mode) or the whole
// array's, shared by the cells and top merges of the dyadic-cell mode.
struct BdCtx {
  void* k0; uint32_t* v0;  // the whole array (virtual position 0)
  void* ks; uint32_t* vs;  // the F scratch blocks
  uint32_t n, NB, P, F;
  uint32_t *Tin, *Tout, *inv, *pool, *remain, *dirty, *didx, *dlist, *first_tile, *cplists;
  void* bstate;
  void* bdesc;
  uint32_t bdesc_cap;
  uint32_t cap() const { return NB + F + 8; }  // the pool ring (NP entries)
};

static BdCtx ctx_of_work(const Work& w, void* k0, uint32_t* v0) {
  BdCtx C;
  C.k0 = k0; C.v0 = v0; C.ks = w.k1; C.vs = w.v1;
  C.n = w.n; C.NB = w.NB; C.P = w.P; C.F = w.F;
  C.Tin = w.Tin; C.Tout = w.Tout; C.inv = w.inv; C.pool = w.pool; C.remain = w.remain; C.dirty = w.dirty;
  C.didx = w.didx; C.dlist = w.dlist; C.first_tile = w.first_tile; C.cplists = w.cplists;
  C.bstate = w.bstate; C.bdesc = w.bdesc; C.bdesc_cap = w.bdesc_cap;
  return C;
}

template <int KT>
static BdMem<KT> bd_mem(const BdCtx& C) {
  using K = typename KeyTraits<KT>::K;
  BdMem<KT> M;
  M.k0 = (K*)C.k0; M.v0 = C.v0; M.ks = (K*)C.ks; M.vs = C.vs;
  M.NB = C.NB; M.P = C.P; M.n = C.n; M.has_partial = (C.n % C.P) != 0;
  M.lg = 0;
  while ((1u << M.lg) < C.P) ++M.lg;
  return M;
}

static vmps_status_t bd_init(const BdCtx& C, cudaStream_t s) {
  LAUNCH(k_bd_init, grid_for(C.cap()), 256, 0, s, (BdState*)C.bstate, C.pool, C.cap(), C.Tin, C.inv, C.NB, C.F,
         C.dirty);
  return VMPS_OK;
}

static vmps_status_t bd_check(const BdCtx& C, cudaStream_t s, const char* what) {
  BdState hs;
  VMPS_CK(cudaMemcpyAsync(&hs, C.bstate, sizeof(hs), cudaMemcpyDeviceToHost, s));
  VMPS_CK(cudaStreamSynchronize(s));
  if (hs.err == 2) { g_err = "internal: bounded tile capacity"; return VMPS_ERR_INTERNAL; }
  if (hs.err) { g_err = std::string("scratch budget too small for the bounded ") + what; return VMPS_ERR_BUDGET; }
  return launch_check();
}

// Level passes p_hi .. p_lo over the runs of w (positions relative to `base`
// in the whole array; made absolute here), restricted to the blocks they
// touch.  fuse_z: nodes of at most this size belong to the leaf stage.
template <int KT, bool HV>
static vmps_status_t bd_levels(const BdCtx& C, const Work& w, uint64_t base, int p_hi, int p_lo, uint32_t fuse_z,
                               cudaStream_t s) {
  if (p_lo > p_hi) return VMPS_OK;
  const BdMem<KT> M = bd_mem<KT>(C);
  BdState* st = (BdState*)C.bstate;
  const unsigned g = grid_for(w.rmax);
  const uint32_t vb0 = (uint32_t)(base / C.P);
  const uint32_t vb1 = (uint32_t)std::min<uint64_t>(C.NB, (base + w.n + C.P - 1) / C.P);
  const uint32_t nbr = vb1 - vb0;
  const unsigned gNB = grid_for(nbr + 8);
  BdTile* desc = (BdTile*)C.bdesc;
  if (base) LAUNCH(k_rs_add_base, g, 256, 0, s, w.run_start, w.scalars, (uint32_t)base);
  // level kernel: persistent grid, shared memory for the block's inputs and outputs
  const int ds = dev_slot();
  static int lv_grid[MAX_DEV][3][2][16] = {};  // by log2 P
  uint32_t lp = 0;
  while ((1u << lp) < C.P) ++lp;
  const size_t lsm = bd_level_smem<KT, HV>(C.P);
  if (!lv_grid[ds][KT][HV][lp]) {
    VMPS_CK(cudaFuncSetAttribute(k_bd_level<KT, HV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)bd_level_smem<KT, HV>(DEFAULT_TOUT)));
    int per_sm = 0;
    VMPS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bd_level<KT, HV>, BD_THREADS, lsm));
    lv_grid[ds][KT][HV][lp] = nsm() * std::max(per_sm, 1);
  }
  const unsigned glv = (unsigned)lv_grid[ds][KT][HV][lp];
  const unsigned gfix = nsm() * 4;
  // highest power first; no host synchronisation: every kernel reads the
  // level's sizes from device memory
  // the call's level schedule: non-fused nodes bucketed by power (stable),
  // tile counts of every node, once
  const uint32_t nlt = (w.rmax + BD_LVL_TILE) / BD_LVL_TILE;
  LAUNCH(k_lvl_hist, nlt, BD_LVL_TILE, 0, s, w.run_start, w.scalars, w.power, w.seg_l, w.seg_r, fuse_z, nlt,
         w.lvl_hist);
  scan_u32(w.lvl_hist, w.lvl_hscan, BD_LVL_BINS * nlt + 1, w.scan_tmp, s);
  LAUNCH(k_lvl_scatter, nlt, BD_LVL_TILE, 0, s, w.run_start, w.scalars, w.power, w.seg_l, w.seg_r, fuse_z, nlt,
         w.lvl_hscan, w.blnodes);
  LAUNCH(k_bd_tile_counts, g, 256, 0, s, w.run_start, w.seg_l, w.seg_r, w.blnodes, w.lvl_hscan, nlt, C.P, C.n,
         w.rmax, w.bcnt);
  scan_u32(w.bcnt, w.btoff, w.rmax + 1, w.scan_tmp, s);
  for (int p = p_hi; p >= p_lo; --p) {
    // tile descriptors + dirty flags (the level's slice of the schedule read
    // on the device), dirty list, level pass, commit: 4 launches per pass on
    // block ranges up to BD_SMALL_MAX, the scan launches above that
    LAUNCH(k_bd_tile_desc<KT>, gfix, 256, 0, s, M, C.Tin, w.run_start, w.seg_l, w.seg_r, w.blnodes, w.lvl_hscan, nlt,
           p, w.btoff, C.bdesc_cap, st, desc, w.bm, vb0, C.dirty);
    if (nbr <= BD_SMALL_MAX) {
      LAUNCH((k_bd_dirty_small<KT>), 1, BD_SMALL_THREADS, 0, s, M, desc, w.bm, C.dirty, C.didx, vb0, nbr, C.dlist,
             C.first_tile, C.remain, w.bD);
    } else {
      scan_u32(C.dirty, C.didx, nbr + 1, w.scan_tmp, s);
      LAUNCH((k_bd_dirty_list<KT>), std::max(gNB, gfix), 256, 0, s, M, desc, w.bm, C.dirty, C.didx, vb0, nbr,
             C.dlist, C.first_tile, C.remain, w.bD);
    }
    LAUNCH((k_bd_level<KT, HV>), glv, BD_THREADS, lsm, s, M, st, desc, w.bm, C.dlist, C.first_tile, w.bD, C.Tin,
           C.Tout, C.pool, C.cap(), C.remain);
    LAUNCH(k_bd_commit, gNB, 256, 0, s, st, C.dlist, w.bD, C.Tout, C.Tin, C.inv, C.dirty, vb0);
  }
  return VMPS_OK;
}

// Final Copy: permute the blocks into physical order (one cooperative kernel).
template <int KT, bool HV>
static vmps_status_t bd_copy(const BdCtx& C, cudaStream_t s) {
  BdState* st = (BdState*)C.bstate;
  LAUNCH(k_bd_ring_to_stack, 1, 1024, 0, s, st, C.pool, C.cap(), C.Tout);
  LAUNCH(k_bd_inverse, grid_for(C.NB + C.F), 256, 0, s, C.Tin, C.NB, C.NB + C.F, C.inv);
  LAUNCH(k_bd_inverse2, grid_for(C.NB + 8), 256, 0, s, C.Tin, C.NB, C.inv);
  VMPS_CK(cudaMemsetAsync(&st->copy_q, 0, 4, s));
  const int ds = dev_slot();
  static bool copy_attr[MAX_DEV][3][2] = {};
  if (!copy_attr[ds][KT][HV]) {
    int per_sm = 0;
    VMPS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bd_copy_all<KT, HV>, BD_CP_THREADS, 0));
    if (per_sm < 1) { g_err = "internal: Copy kernel not resident"; return VMPS_ERR_INTERNAL; }
    copy_attr[ds][KT][HV] = true;
  }
  BdMem<KT> Mc = bd_mem<KT>(C);
  uint32_t* Tin = C.Tin;
  uint32_t* inv = C.inv;
  uint32_t* pool = C.pool;
  uint32_t* lists = C.cplists;
  void* args[] = {&Mc, &st, &Tin, &inv, &pool, &lists};
  VMPS_CK(cudaLaunchCooperativeKernel((const void*)k_bd_copy_all<KT, HV>, dim3(nsm()), dim3(BD_CP_THREADS), args, 0,
                                      s));
  ++g_nl;
  return VMPS_OK;
}

// Bring virtual block b back to its own physical block (dyadic-cell mode:
// the first block of a range that is read in place, after the previous range
// rewrote it through the table).
template <int KT, bool HV>
static vmps_status_t bd_home(const BdCtx& C, uint32_t b, uint32_t* d_slot, cudaStream_t s) {
  if (b >= C.NB) return VMPS_OK;
  BdState* st = (BdState*)C.bstate;
  VMPS_CK(cudaMemsetAsync(d_slot, 0xFF, 4, s));
  LAUNCH(k_bd_find_free, nsm() * 2, 256, 0, s, st, C.Tin, C.pool, C.cap(), b, d_slot);
  LAUNCH((k_bd_home<KT, HV>), 1, 512, 0, s, bd_mem<KT>(C), st, C.Tin, C.inv, C.pool, C.cap(), b, d_slot);
  return VMPS_OK;
}

template <bool HV>
static vmps_status_t bounded_stats(const Work& w, vmps_stats_t* st, cudaStream_t s) {
  if (g_prof && g_prof_host) {
    VMPS_CK(cudaMemcpyAsync(g_prof_host, w.counters, 24, cudaMemcpyDeviceToHost, s));
    g_prof_wbytes = (int)(key_bytes(w.kt) + (HV ? 4 : 0));
  }
  if (!st) return VMPS_OK;
  uint32_t sc[SC_COUNT];
  unsigned long long ct[8];
  BdState hs;
  VMPS_CK(cudaMemcpyAsync(sc, w.scalars, sizeof(sc), cudaMemcpyDeviceToHost, s));
  VMPS_CK(cudaMemcpyAsync(ct, w.counters, sizeof(ct), cudaMemcpyDeviceToHost, s));
  VMPS_CK(cudaMemcpyAsync(&hs, w.gt_ctx ? ((const BdCtx*)w.gt_ctx)->bstate : w.bstate, sizeof(hs),
                          cudaMemcpyDeviceToHost, s));
  VMPS_CK(cudaStreamSynchronize(s));
  memset(st, 0, sizeof(*st));
  st->n = w.n;
  st->runs = sc[SC_RUNS];
  st->merges = sc[SC_RUNS] ? sc[SC_RUNS] - 1 : 0;
  st->merge_cost_M = ct[0];
  st->fused_M = ct[1];
  st->reversed_elems = sc[SC_REVERSED];
  st->extended_runs = sc[SC_EXTENDED];
  st->max_power = sc[SC_MAXPOW];
  st->minrun = w.minrun;
  st->block_elems = w.P;
  st->rounds = hs.rounds;
  st->peak_extra_device_bytes = w.used_bytes;
  st->scratch_bytes = w.scratch_bytes;
  st->metadata_bytes = w.used_bytes - w.scratch_bytes;
  return VMPS_OK;
}

static bool kernel_attrs_set[MAX_DEV][3][2] = {};

template <int KT, bool HV>
static vmps_status_t sort_impl(const Work& w, void* keys, uint32_t* vals, cudaStream_t s,
                               vmps_stats_t* st, const GivenRuns* G = nullptr) {
  using K = typename KeyTraits<KT>::K;
  prof_reset();
  const double g_bdt_front = bd_now(s);
  NvtxRange nv_sort("vmps_sort");
  NvtxRange nv_plan("vmps_plan");
  g_prof_mark[0] = prof_event(s);
  vmps_status_t rc = G ? front_half_given(w, *G, s) : front_half<KT>(w, keys, s);
  if (rc != VMPS_OK) return rc;
  const uint32_t* dep = w.dep[0];
  const unsigned g = grid_for(w.rmax);
  VMPS_CK(cudaMemsetAsync(w.level_cnt, 0, (LEVEL_SLOTS + 1) * 4, s));
  VMPS_CK(cudaMemsetAsync(w.level_fill, 0, (LEVEL_SLOTS + 1) * 4, s));
  LAUNCH(k_class_nodes, g, 256, 0, s, w.run_start, w.scalars, w.counters, w.power, w.seg_l, w.seg_r, w.parent,
         dep, w.fuse_z, w.unit_end, w.unit_par, w.level_cnt, w.fuse2);
  LAUNCH(k_class_runs, g, 256, 0, s, w.run_start, w.run_kind, w.scalars, w.power, w.seg_l, w.seg_r, dep,
         w.fuse_z, w.rmax, w.unit_flag, w.long_flag, w.unit_end, w.unit_par, w.long_par, w.fuse2);
  if (w.fuse2) {
    VMPS_CK(cudaMemsetAsync(w.lchild, 0, ((size_t)w.rmax + 2) * 4, s));
    VMPS_CK(cudaMemsetAsync(w.rchild, 0, ((size_t)w.rmax + 2) * 4, s));
    LAUNCH(k_child_map, g, 256, 0, s, w.run_start, w.scalars, w.seg_l, w.seg_r, w.parent, w.fuse_z, w.lchild,
           w.rchild);
  }
  scan_u32(w.unit_flag, w.unit_idx, w.rmax + 1, w.scan_tmp, s);
  scan_u32(w.long_flag, w.long_idx, w.rmax + 1, w.scan_tmp, s);
  LAUNCH(k_compact, g, 256, 0, s, w.run_start, w.scalars, w.unit_flag, w.unit_idx, w.long_flag, w.long_idx,
         w.unit_end, w.unit_par, w.long_par, w.units, w.longs, w.long_chunks, w.bounded ? 0u : 1u);
  LAUNCH(k_zero_tail, g, 256, 0, s, w.long_chunks, w.scalars, (int)SC_LONG, w.rmax);
  scan_u32(w.long_chunks, w.long_off, w.rmax + 1, w.scan_tmp, s);
  LAUNCH(k_level_scan, 1, 32, 0, s, w.level_cnt, w.level_start, w.scalars);
  if (!w.bounded) {
    LAUNCH(k_level_scatter, g, 256, 0, s, w.run_start, w.scalars, w.power, w.seg_l, w.seg_r, w.fuse_z,
           w.level_start, w.level_fill, w.lnodes, dep, w.fuse2);
    LAUNCH(k_level_tiles, g, 256, 0, s, w.run_start, w.scalars, w.seg_l, w.seg_r, w.lnodes, w.tout, w.rmax,
           w.ltiles_cnt);
    scan_u32(w.ltiles_cnt, w.ltiles, w.rmax + 1, w.scan_tmp, s);
    LAUNCH(k_level_tile_off, 1, 128, 0, s, w.level_start, w.ltiles, w.level_tile);
  }
  rc = launch_check();
  if (rc != VMPS_OK) return rc;
  g_prof_mark[1] = prof_event(s);
  nv_plan.end();

  // leaf engine
  NvtxRange nv_leaf("vmps_leaf");
  K* k0 = (K*)keys;
  K* k1 = (K*)w.k1;
  uint32_t* v0 = vals;
  uint32_t* v1 = w.v1;
  const size_t lsm = leaf_smem_bytes<KT>(HV);
  const size_t lsm2 = leaf_smem_bytes<KT, LEAF_SMALL>(HV);
  const size_t rsm = LeafRadixSmem<KT>::BYTES;
  const int ds = dev_slot();
  if (!kernel_attrs_set[ds][KT][HV]) {
    VMPS_CK(cudaFuncSetAttribute(k_leaf_sort<KT, HV, LEAF_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)lsm));
    VMPS_CK(cudaFuncSetAttribute(k_leaf_sort<KT, HV, LEAF_SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)lsm2));
    VMPS_CK(cudaFuncSetAttribute(k_leaf_radix<KT, HV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
    kernel_attrs_set[ds][KT][HV] = true;
  }
  // a batch = consecutive touching units starting in one window of Zb
  // positions; units are <= Z long, so a batch spans < Zb + Z <= LEAF_CAP
  // elements and fills most of the CTA.  Batches <= windows + long leaves.
  const uint32_t zb = leaf_zb(w.fuse_z, w.bounded);
  const uint32_t nbatch = w.bcap;
  LAUNCH(k_batch_flags, g, 256, 0, s, w.units, w.scalars, zb, w.rmax, w.unit_flag);
  scan_u32(w.unit_flag, w.unit_idx, w.rmax + 1, w.scan_tmp, s);
  LAUNCH(k_batch_first, grid_for(nbatch + 1), 256, 0, s, w.unit_flag, w.unit_idx, w.scalars, nbatch, w.batch_first);
  if (g_leaf_radix)
    LAUNCH((k_leaf_radix<KT, HV>), nbatch, LEAF_THREADS, rsm, s, k0, v0, k1, v1, w.units, w.batch_first);
  else {
    LAUNCH((k_leaf_sort<KT, HV, LEAF_SMALL>), nsm() * 2 * leaf_minb<KT>(), LEAF_SMALL, lsm2, s, k0, v0, k1, v1,
           w.units, w.batch_first, w.scalars);
    if (zb + w.fuse_z - 1 > (uint32_t)LEAF_SMALL_CAP)  // some batch may exceed the half-size CTA
      LAUNCH((k_leaf_sort<KT, HV, LEAF_THREADS>), nsm() * leaf_minb<KT>(), LEAF_THREADS, lsm, s, k0, v0, k1, v1,
             w.units, w.batch_first, w.scalars);
  }
  LAUNCH((k_long_leaves<KT, HV>), nsm() * VMPS_LONG_MINB, 256, 0, s, k0, v0, k1, v1, w.longs, w.long_off, w.scalars,
         LONG_CHUNK);
  rc = launch_check();
  if (rc != VMPS_OK) return rc;
  g_prof_mark[2] = prof_event(s);
  nv_leaf.end();
  NvtxRange nv_merge("vmps_merge");

  // level merges, highest power first (children before parents, F3)
  double lg = std::log2(2.0 * (double)(G && G->global() ? G->n_glob : (uint64_t)w.n) / (double)w.fuse_z);
  int p_hi = (int)std::ceil(lg) + 1;
  if (p_hi > LEVEL_SLOTS - 2) p_hi = LEVEL_SLOTS - 2;
  if (p_hi < 1) p_hi = 1;
  int p_lo = 1;
  if (G && w.bounded && G->p_min > 0) {
    p_lo = G->p_min;
  } else if (G && w.bounded) {  // given runs: only the powers their boundaries carry
    const uint64_t N = G->gpos ? G->n_glob : (uint64_t)w.n;
    auto pos = [&](uint32_t i) -> uint64_t { return G->gpos ? G->gpos[i] : (uint64_t)G->rel[i]; };
    uint32_t mn = 0xFFFFFFFFu, mx = 0;
    for (uint32_t i = 1; i < G->r; ++i) {
      const uint32_t pw = host_power(N, pos(i - 1), pos(i), pos(i + 1));
      mn = std::min(mn, pw);
      mx = std::max(mx, pw);
    }
    p_hi = std::min<int>(p_hi, (int)mx);
    p_lo = G->r > 1 ? (int)mn : p_hi + 1;
  }
  if (w.bounded) {
    bd_add(3, g_bdt_front, s);
    double t0 = bd_now(s);
    if (w.gt_ctx) {  // a cell of the dyadic-cell mode: the whole array's table, no Copy
      const BdCtx& C = *(const BdCtx*)w.gt_ctx;
      // no host synchronisation per cell: errors stay in the shared state
      // (every level kernel stops on them) and the caller checks it once
      rc = bd_levels<KT, HV>(C, w, w.gt_base, p_hi, p_lo, w.fuse_z, s);
      bd_add(1, t0, s);
      if (rc != VMPS_OK) return rc;
      return bounded_stats<HV>(w, st, s);
    }
    const BdCtx C = ctx_of_work(w, k0, v0);
    rc = bd_init(C, s);
    if (rc == VMPS_OK) rc = bd_levels<KT, HV>(C, w, 0, p_hi, p_lo, w.fuse_z, s);
    if (rc == VMPS_OK) rc = bd_check(C, s, "mode");
    bd_add(1, t0, s);
    t0 = bd_now(s);
    if (rc == VMPS_OK) rc = bd_copy<KT, HV>(C, s);
    if (rc == VMPS_OK) rc = bd_check(C, s, "Copy");
    bd_add(2, t0, s);
    if (rc != VMPS_OK) return rc;
    if (bd_trace() && !G) {  // one-piece bounded sort
      static const char* nm[4] = {"-", "levels", "copy", "front+leaf"};
      for (int i = 1; i < 4; ++i) fprintf(stderr, "vmps bd trace: %-10s %9.1f ms  %ld\n", nm[i], g_bdt.t[i], g_bdt.n[i]);
      memset(&g_bdt, 0, sizeof(g_bdt));
    }
    g_prof_mark[3] = prof_event(s);
    return bounded_stats<HV>(w, st, s);
  }
  if (w.fuse2) {
    using SM4 = Merge4Smem<KT, HV>;
    static int occ4_t[MAX_DEV][3][2] = {};
    auto& occ4 = occ4_t[ds];
    if (!occ4[KT][HV]) {
      VMPS_CK(cudaFuncSetAttribute(k4_merge_level<KT, HV, M4_KQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)SM4::BYTES));
      int occ = 0;
      VMPS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k4_merge_level<KT, HV, M4_KQ>, M4_THREADS,
                                                            SM4::BYTES));
      occ4[KT][HV] = occ > 0 ? occ : 1;
    }
    const unsigned gm4 = (unsigned)(nsm() * occ4[KT][HV]);
    // warp-per-tile partition for small levels: up to 16,384 tiles while the
    // keys stay near the L2 (its probes are many but parallel), 4,096 beyond;
    // measured at cfg1-5
    const uint32_t desc_warp_max =
        !VMPS_DESC4_WARP ? 0u : (uint64_t)w.n * sizeof(K) <= (512ull << 20) ? DESC4_WARP_MAX : VMPS_DESC4_WARP_MAX_BIG;
    NodeRuns* nr = (NodeRuns*)w.nr4;
    TileDesc4* t4 = (TileDesc4*)w.tiles4;
    for (int p = p_hi; p >= 1; --p) {
      int e0 = prof_event(s);
      LAUNCH(k4_node_runs, grid_for(w.n4cap), 256, 0, s, w.run_start, w.seg_l, w.seg_r, dep, w.lchild, w.rchild,
             w.lnodes, w.level_start, p, nr);
      LAUNCH(k4_desc<KT>, (std::max<uint32_t>(w.part_cap / 4, std::min<uint32_t>(w.part_cap, 4 * DESC4_SERIAL_MIN)) + 256) / 256, 256, 0, s, k0, k1, nr, w.ltiles, w.level_start,
             w.level_tile, p, w.tout, t4, desc_warp_max);
      if (desc_warp_max)
        LAUNCH(k4_desc_warp<KT>, (32u * std::min<uint32_t>(w.part_cap, desc_warp_max) + 255) / 256, 256, 0, s, k0, k1,
               nr, w.ltiles, w.level_start, w.level_tile, p, w.tout, t4, desc_warp_max);
      int e1 = prof_event(s);
      LAUNCH((k4_merge_level<KT, HV, M4_KQ>), gm4, M4_THREADS, SM4::BYTES, s, k0, v0, k1, v1, t4, nr, w.level_tile, p);
      ++g_nl_merge;
      int e2 = prof_event(s);
      if (g_prof && e0 >= 0 && e2 >= 0 && g_prof_nm < 128) {
        g_prof_part[g_prof_np][0] = e0; g_prof_part[g_prof_np][1] = e1; g_prof_np++;
        g_prof_lvl[g_prof_nm][0] = e1; g_prof_lvl[g_prof_nm][1] = e2; g_prof_nm++;
      }
    }
  } else {
  using SM = MergeSmem<KT, HV>;
  static int merge_occ_t[MAX_DEV][3][2] = {};
  auto& merge_occ = merge_occ_t[ds];
  if (!merge_occ[KT][HV]) {
    VMPS_CK(cudaFuncSetAttribute(k_merge_level<KT, HV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SM::BYTES));
    int occ = 0;
    VMPS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_merge_level<KT, HV>, MERGE_BLOCK, SM::BYTES));
    merge_occ[KT][HV] = occ > 0 ? occ : 1;
  }
  const unsigned gm = (unsigned)(nsm() * merge_occ[KT][HV]);
  TileDesc* desc = (TileDesc*)w.desc;
  for (int p = p_hi; p >= 1; --p) {
    int e0 = prof_event(s);
    LAUNCH(k_tile_desc<KT>, (w.part_cap / DESC_CHUNK + 256) / 256, 256, 0, s, k0, k1, w.run_start, w.seg_l, w.seg_r, dep, w.lnodes,
           w.ltiles, w.level_start, w.level_tile, p, w.tout, desc, w.part_cap, w.scalars);
    int e1 = prof_event(s);
    LAUNCH((k_merge_level<KT, HV>), gm, MERGE_BLOCK, SM::BYTES, s, k0, v0, k1, v1, desc, w.level_tile, p,
           w.tout, w.part_cap);
    ++g_nl_merge;
    int e2 = prof_event(s);
    if (g_prof && e0 >= 0 && e2 >= 0 && g_prof_nm < 128) {
      g_prof_part[g_prof_np][0] = e0; g_prof_part[g_prof_np][1] = e1; g_prof_np++;
      g_prof_lvl[g_prof_nm][0] = e1; g_prof_lvl[g_prof_nm][1] = e2; g_prof_nm++;
    }
  }
  }  // level-by-level merges
  LAUNCH(k_check_levels, 1, 32, 0, s, w.level_cnt, p_hi, w.scalars, w.fuse2 ? w.level_tile : nullptr, w.part_cap);
  if (!st) LAUNCH(k_error_guard, 1, 1, 0, s, w.scalars);  // with h_stats: VMPS_ERR_INTERNAL below
  rc = launch_check();
  if (rc != VMPS_OK) return rc;
  g_prof_mark[3] = prof_event(s);
  if (g_prof && g_prof_host) {
    VMPS_CK(cudaMemcpyAsync(g_prof_host, w.counters, 24, cudaMemcpyDeviceToHost, s));
    g_prof_wbytes = (int)(key_bytes(w.kt) + (HV ? 4 : 0));
  }

  if (st) {
    uint32_t sc[SC_COUNT];
    unsigned long long ct[8];
    uint32_t lc[LEVEL_SLOTS + 1];
    VMPS_CK(cudaMemcpyAsync(sc, w.scalars, sizeof(sc), cudaMemcpyDeviceToHost, s));
    VMPS_CK(cudaMemcpyAsync(ct, w.counters, sizeof(ct), cudaMemcpyDeviceToHost, s));
    VMPS_CK(cudaMemcpyAsync(lc, w.level_cnt, sizeof(lc), cudaMemcpyDeviceToHost, s));
    VMPS_CK(cudaStreamSynchronize(s));
    if (sc[SC_ERROR]) {
      g_err = sc[SC_ERROR] == 2 ? "internal: tile descriptor capacity exceeded"
                                : "internal: a non-fused node has a power above the launched levels";
      return VMPS_ERR_INTERNAL;
    }
    memset(st, 0, sizeof(*st));
    st->n = w.n;
    st->runs = sc[SC_RUNS];
    st->merges = sc[SC_RUNS] ? sc[SC_RUNS] - 1 : 0;
    st->merge_cost_M = ct[0];
    st->fused_M = ct[1];
    st->hbm_merge_elems = ct[2];
    st->reversed_elems = sc[SC_REVERSED];
    st->extended_runs = sc[SC_EXTENDED];
    st->max_power = sc[SC_MAXPOW];
    uint32_t lv = 0;
    for (int p = 0; p <= LEVEL_SLOTS; ++p) lv += lc[p] ? 1 : 0;
    st->levels_executed = lv;
    st->minrun = w.minrun;
    st->peak_extra_device_bytes = w.used_bytes;
    st->scratch_bytes = (uint64_t)w.n * (key_bytes(w.kt) + (HV ? 4 : 0));
    st->metadata_bytes = w.used_bytes - st->scratch_bytes;
  }
  return VMPS_OK;
}

}  // namespace vmps

using namespace vmps;

namespace vmps {
// ---- distributed plan building blocks ----
// Run detection of one shard of a larger array: the chain's entry state at
// the shard start comes from the caller (composition of the previous shards'
// tables), END only at the global end (n_end), descent bits across the shard
// edges from *d_prev (previous shard's last key) and d_halo (the next keys).
template <int KT>
static vmps_status_t shard_front(const Work& w, const void* keys, uint32_t n_end, const void* d_prev,
                                 const void* d_halo, uint32_t n_halo, cudaStream_t s) {
  using K = typename KeyTraits<KT>::K;
  vmps_status_t arc = chain_attrs();
  if (arc != VMPS_OK) return arc;
  VMPS_CK(cudaMemsetAsync(w.scalars, 0, SC_COUNT * 4, s));
  LAUNCH(k_runs_tables<KT>, w.ntiles, 128, 0, s, (const K*)keys, w.n, w.minrun, w.ns, w.bits, w.tile_tab, n_end,
         (const K*)d_prev, (const K*)d_halo, n_halo);
  const size_t sm32 = (size_t)CHAIN_G * w.ns * 4, sm64 = (size_t)CHAIN_G * w.ns * 8;
  for (int l = 0; l < w.chain_levels; ++l) {
    if (l == 0)
      LAUNCH(k_chain_compose<uint32_t>, w.chain_m[1], 256, sm32, s, w.tile_tab, w.chain_m[0], w.ns, w.chain_tab[0]);
    else
      LAUNCH(k_chain_compose<uint64_t>, w.chain_m[l + 1], 256, sm64, s, w.chain_tab[l - 1], w.chain_m[l], w.ns,
             w.chain_tab[l]);
  }
  return launch_check();
}

// Shard-local u32 run starts -> global u64 positions.
__global__ void k_shard_starts(const uint32_t* __restrict__ local, uint64_t count, uint64_t offset,
                               uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = offset + local[i];
}

template <int KT>
static vmps_status_t shard_dispatch_front(const Work& w, const void* keys, uint32_t n_end, const void* d_prev,
                                          const void* d_halo, uint32_t n_halo, cudaStream_t s) {
  return shard_front<KT>(w, keys, n_end, d_prev, d_halo, n_halo, s);
}

}  // namespace vmps

static vmps_status_t check_common(const void* keys, const void* vals, uint64_t n, vmps_key_t kt) {
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) {
    g_err = "unknown key type";
    return VMPS_ERR_INVALID_ARG;
  }
  if (n > VMPS_MAX_N) {
    g_err = "n > VMPS_MAX_N (2^32 - 2^16) is not supported";
    return VMPS_ERR_INVALID_ARG;
  }
  if (n > 1 && !keys) {
    g_err = "keys is NULL";
    return VMPS_ERR_INVALID_ARG;
  }
  if (((uintptr_t)keys & 15) || ((uintptr_t)vals & 15)) {
    g_err = "keys/vals must be 16-byte aligned";
    return VMPS_ERR_INVALID_ARG;
  }
  return VMPS_OK;
}

extern "C" {

// Dyadic-cell scratch-bounded mode (large n): Alg. 1 run over
// cells.  With q = ceil(log2(n / CELL)), every node of power > q lies inside
// one dyadic cell of level q of the midpoint space (its runs' midpoints share
// the node's cell of level p - 1 >= q), so the runs whose midpoints fall in a
// cell form one subtree of the whole plan, and the boundaries between cells
// carry the powers <= q.  The array is scanned left to right in detection
// chunks (run-detection transfer table + run emission per chunk, the chain
// state carried across chunks, original edge keys kept aside, the runs kept in
// a device ring); each cell, once its last run's end is known, is sorted by
// the bounded engine from its runs with the global powers (exactly the whole
// plan's subtree), and the cell results go through Alg. 1's stack with the
// boundary powers computed from the original runs (each pop one level pass
// of a single node).  Cells and pops write through ONE block table of the
// whole array (the paper's page table): a range read in place (a
// cell's leaves, a detection chunk) first brings its first block home, the
// only block an earlier range can have rewritten; one Copy at the end.  The
// executed merges are exactly Alg. 1's plan (M equal to the one-piece mode),
// while the device metadata scales with a cell (runs with midpoints in it
// <= CELL / minrun + 2) plus n / P block-table entries instead of n / minrun
// run entries: 3.4 GB -> 93 MB at cfg5 (2^30, CELL = 2^23).
#ifndef VMPS_BD_CHUNK
#define VMPS_BD_CHUNK (1u << 23)
#endif
#ifndef VMPS_BD_DET
#define VMPS_BD_DET (1u << 23)  // run-detection chunk of the dyadic-cell mode (elements)
#endif
static uint64_t g_bd_chunk = VMPS_BD_CHUNK;  // cell size target (test hook vmps_test_set_bd_chunk)
static bool bd_chunked(uint64_t n, int64_t scratch, int hv) { return scratch >= 0 && hv >= 0 && n > 2 * g_bd_chunk; }
static uint32_t bd_cell_level(uint64_t n) {
  uint32_t q = 0;
  while ((n >> q) > g_bd_chunk) ++q;
  return q;
}
struct CellLayout {
  size_t det_ws, det_out, sort_ws, gt, total;
  uint32_t det;    // detection chunk (elements)
  uint32_t rcell;  // runs of one cell, at most
  uint64_t ring;   // device ring of unconsumed runs (entries)
};
// The whole array's block table and element scratch (dyadic-cell mode).
static size_t carve_gt(const Cfg& c, uint32_t rcell, char* base, BdCtx* C) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> void* {
    void* p = base ? (void*)(base + off) : nullptr;
    off += align_up(bytes);
    return p;
  };
  BdCtx t{};
  t.n = (uint32_t)c.n;
  t.P = c.P;
  t.F = c.F;
  t.NB = (uint32_t)((c.n + c.P - 1) / c.P);
  const size_t se = (size_t)c.F * c.P;
  t.ks = take(se * key_bytes(c.kt));
  t.vs = c.hv ? (uint32_t*)take(se * 4) : nullptr;
  const size_t NBp = (size_t)t.NB + 8, NP = (size_t)t.NB + c.F + 8;
  t.Tin = (uint32_t*)take(NBp * 4);
  t.Tout = (uint32_t*)take(NBp * 4);
  t.inv = (uint32_t*)take(NP * 4);
  t.pool = (uint32_t*)take(NP * 4);
  t.remain = (uint32_t*)take(NBp * 4);
  t.dirty = (uint32_t*)take(NBp * 4);
  t.didx = (uint32_t*)take(NBp * 4);
  t.dlist = (uint32_t*)take(NBp * 4);
  t.first_tile = (uint32_t*)take(NBp * 4);
  // a level's tiles: the nodes of one power are disjoint and hold >= 2 runs
  // each (<= rcell / 2 nodes); a node spans its blocks (+1 shared with a
  // neighbour) plus <= 2 gap tiles: <= NB + 1.5 rcell
  t.bdesc_cap = t.NB + rcell + rcell / 2 + 16;
  t.bdesc = take((size_t)t.bdesc_cap * sizeof(BdTile));
  t.bstate = take(sizeof(BdState));
  t.cplists = (uint32_t*)take((size_t)2 * BD_CP_LIST * 4);
  take(64);  // bd_home's slot
  if (C) *C = t;
  return off;
}
static CellLayout bd_cell_layout(uint64_t n, int kt, int hv, int64_t scratch) {
  CellLayout L{};
  Cfg c0 = make_cfg(n, kt, hv, scratch);
  L.det = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(g_bd_chunk, VMPS_BD_DET), n);
  size_t b = 0;
  vmps_shard_workspace_bytes(L.det, (vmps_key_t)kt, c0.minrun, &b);
  L.det_ws = align_up(b);
  const uint64_t rdet = L.det / std::max<uint32_t>(c0.minrun, 1) + 4;
  // a cell's sort: its runs (<= cell / minrun + 2); the block table is the whole array's
  L.rcell = (uint32_t)(((n >> bd_cell_level(n)) + 1) / std::max<uint32_t>(c0.minrun, 1) + 4);
  L.ring = L.rcell + 2 * rdet + 16;  // unconsumed runs: an open cell's and two detection chunks'
  L.det_out = align_up(rdet * 8) + align_up(rdet + 16) + align_up((size_t)3 * 64 * 8) + align_up(64) +
              align_up(L.ring * 8) + align_up(L.ring);
  Cfg cs = make_cfg(n, kt, hv, scratch);
  cs.given_runs = L.rcell;
  cs.gt_nb = (uint32_t)((n + c0.P - 1) / c0.P);
  L.sort_ws = align_up(carve(cs, nullptr, nullptr));
  L.gt = align_up(carve_gt(c0, L.rcell, nullptr, nullptr));
  L.total = L.det_ws + L.det_out + L.sort_ws + L.gt + 256;
  return L;
}

vmps_status_t vmps_workspace_bytes(uint64_t n, vmps_key_t kt, int has_vals, int64_t scratch_elems,
                                   size_t* h_bytes) {
  if (!h_bytes) return VMPS_ERR_INVALID_ARG;
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) return VMPS_ERR_INVALID_ARG;
  if (n > VMPS_MAX_N) return VMPS_ERR_INVALID_ARG;
  if (n <= 1) { *h_bytes = 256; return VMPS_OK; }
  const int hv = has_vals < 0 ? -1 : (has_vals ? 1 : 0);
  if (bd_chunked(n, scratch_elems, hv)) { *h_bytes = bd_cell_layout(n, kt, hv, scratch_elems).total + 256; return VMPS_OK; }
  Cfg c = make_cfg(n, kt, hv, scratch_elems);
  *h_bytes = carve(c, nullptr, nullptr) + 256;
  return VMPS_OK;
}

}  // extern "C"

static vmps_status_t shard_runs_impl(const void* keys, uint64_t n_local, vmps_key_t kt, uint32_t minrun,
                                     uint32_t n_end, const void* d_prev, const void* d_halo, uint32_t n_halo,
                                     uint32_t entry_state, uint64_t count, uint64_t offset, uint64_t* d_run_start,
                                     uint8_t* d_run_kind, void* ws, size_t ws_bytes, void* stream, bool front_done);

// Pinned host staging of the dyadic-cell mode's detection (per host thread,
// grown on demand): the chain table and one chunk's run starts / kinds.
struct DetHost {
  uint64_t* tab = nullptr;
  uint64_t* rs = nullptr;
  uint8_t* rk = nullptr;
  size_t ntab = 0, nrs = 0;
  ~DetHost() {
    if (tab) cudaFreeHost(tab);
    if (rs) cudaFreeHost(rs);
    if (rk) cudaFreeHost(rk);
  }
  bool reserve(size_t nt, size_t nr) {
    if (nt > ntab) {
      if (tab) cudaFreeHost(tab);
      tab = nullptr;
      if (cudaMallocHost(&tab, nt * 8) != cudaSuccess) { ntab = 0; return false; }
      ntab = nt;
    }
    if (nr > nrs) {
      if (rs) cudaFreeHost(rs);
      if (rk) cudaFreeHost(rk);
      rs = nullptr;
      rk = nullptr;
      if (cudaMallocHost(&rs, nr * 8) != cudaSuccess || cudaMallocHost(&rk, nr) != cudaSuccess) { nrs = 0; return false; }
      nrs = nr;
    }
    return true;
  }
};
static thread_local DetHost g_det_host;

template <int KT, bool HV>
static vmps_status_t sort_bounded_cells(void* keys, uint32_t* vals, uint64_t n, int64_t S, char* base,
                                        cudaStream_t s, vmps_stats_t* st) {
  using K = typename KeyTraits<KT>::K;
  const size_t kb = key_bytes(KT);
  const CellLayout L = bd_cell_layout(n, KT, HV ? 1 : 0, S);
  const Cfg c0 = make_cfg(n, KT, HV ? 1 : 0, S);
  const uint32_t minrun = c0.minrun, ns = 3 * minrun, H = minrun + 8;
  const uint32_t q = bd_cell_level(n);
  const uint32_t NB = (uint32_t)((n + c0.P - 1) / c0.P);
  char* det_ws = base;
  char* det_out = base + L.det_ws;
  char* sort_ws = det_out + L.det_out;
  BdCtx C;
  carve_gt(c0, L.rcell, sort_ws + L.sort_ws, &C);
  C.k0 = keys;
  C.v0 = vals;
  uint32_t* d_slot = (uint32_t*)((char*)C.cplists + align_up((size_t)2 * BD_CP_LIST * 4));
  const uint64_t rdet = L.det / std::max<uint32_t>(minrun, 1) + 4;
  uint64_t* d_rs = (uint64_t*)det_out;
  uint8_t* d_rk = (uint8_t*)(det_out + align_up(rdet * 8));
  uint64_t* d_tab = (uint64_t*)(det_out + align_up(rdet * 8) + align_up(rdet + 16));
  K* d_prev = (K*)(det_out + align_up(rdet * 8) + align_up(rdet + 16) + align_up((size_t)3 * 64 * 8));
  uint64_t* d_ring = (uint64_t*)((char*)d_prev + align_up(64));
  uint8_t* d_ring_kind = (uint8_t*)d_ring + align_up(L.ring * 8);
  uint64_t g_total = 0;  // runs appended to the ring
  vmps_status_t rc = bd_init(C, s);
  if (rc != VMPS_OK) return rc;
  std::vector<uint64_t> R;   // run starts of the unprocessed runs (global; R[0] is run gbase)
  std::vector<uint8_t> RK;   // their kinds
  size_t R0 = 0;             // first unprocessed run
  uint64_t gbase = 0;
  std::vector<uint64_t> tab(ns);
  uint64_t M = 0, runs = 0, rev = 0, ext = 0;
  uint32_t maxp = 0, lv = 0;
  auto cell_of = [&](uint64_t a, uint64_t b) -> uint64_t {  // dyadic cell (level q) of the midpoint of [a, b)
    return (uint64_t)(((unsigned __int128)(a + b) << q) / ((unsigned __int128)2 * n));
  };
  // the least a + b whose cell is after cell c: ceil((c + 1) 2n / 2^q)
  auto cell_end = [&](uint64_t c) -> uint64_t {
    const unsigned __int128 num = (unsigned __int128)(c + 1) * 2 * n;
    return (uint64_t)((num + (((unsigned __int128)1 << q) - 1)) >> q);
  };
  // Alg. 1 over the cell results: segments [a, b) with, for the boundary
  // powers, the first run's end and the last run's start (original runs)
  struct Seg { uint64_t a, b, first_end, last_start; uint32_t pw; };
  std::vector<Seg> stk;
  bool have_curr = false;
  Seg curr{};
  // a top merge [x.a, x.b) (+) [x.b, y.b): one node through the shared table
  auto merge2 = [&](const Seg& x, const Seg& y) -> vmps_status_t {
    const uint64_t len = y.b - x.a;
    M += len;
    const double t0 = bd_now(s);
    Cfg cc = make_cfg(len, KT, HV ? 1 : 0, S);
    cc.given_runs = 2;
    cc.gt_nb = NB;
    Work w;
    if (carve(cc, nullptr, nullptr) > L.sort_ws) { g_err = "internal: top merge workspace"; return VMPS_ERR_INTERNAL; }
    carve(cc, &w, sort_ws);
    // two runs [0, x.b - x.a) [x.b - x.a, len), one node of power 1 (no host copy, no sync)
    LAUNCH(k_bd_top_setup, 1, 64, 0, s, w.run_start, w.seg_l, w.seg_r, w.power, w.scalars,
           (uint32_t)(x.b - x.a), (uint32_t)len);
    vmps_status_t r2 = bd_levels<KT, HV>(C, w, x.a, 1, 1, 0u, s);
    bd_add(6, t0, s);
    return r2;
  };
  auto push_cell = [&](const Seg& nx) -> vmps_status_t {
    if (!have_curr) { curr = nx; have_curr = true; return VMPS_OK; }
    const uint32_t p = host_power(n, curr.last_start, curr.b, nx.first_end);  // Alg. 1 line 6
    maxp = std::max(maxp, p);
    while (!stk.empty() && stk.back().pw >= p) {  // lines 7-9
      vmps_status_t r2 = merge2(stk.back(), curr);
      if (r2 != VMPS_OK) return r2;
      curr = Seg{stk.back().a, curr.b, stk.back().first_end, curr.last_start, 0};
      stk.pop_back();
    }
    curr.pw = p;
    stk.push_back(curr);  // line 10
    curr = nx;            // line 11
    return VMPS_OK;
  };
  // sort the cell made of runs R[R0, R0 + m) (the last ends at end); consume them
  auto do_cell = [&](size_t m, uint64_t end) -> vmps_status_t {
    const double tdc = bd_now(s);
    struct Add { double t0; cudaStream_t s; ~Add() { bd_add(9, t0, s); } } add_dc{tdc, s};
    const uint64_t* Rr = R.data() + R0;
    const uint8_t* RKr = RK.data() + R0;
    const uint64_t a = Rr[0];
    const bool trivial = m == 1 && RKr[0] == 0;  // one ascending run: already sorted
    if (!trivial) {
      const double th = bd_now(s);
      vmps_status_t r2 = bd_home<KT, HV>(C, (uint32_t)(a / c0.P), d_slot, s);  // read in place below
      bd_add(0, th, s);
      if (r2 != VMPS_OK) return r2;
      Cfg cc = make_cfg(end - a, KT, HV ? 1 : 0, S);
      cc.given_runs = (uint32_t)m;
      cc.gt_nb = NB;
      Work w;
      const size_t need = carve(cc, &w, nullptr);
      if (need > L.sort_ws || m > L.rcell) { g_err = "internal: cell workspace"; return VMPS_ERR_INTERNAL; }
      carve(cc, &w, sort_ws);
      w.gt_ctx = &C;
      w.gt_base = a;
      GivenRuns G{nullptr, nullptr, nullptr, n, (uint32_t)m, (int)q + 1};
      G.d_ring = d_ring;
      G.d_ring_kind = d_ring_kind;
      G.ring_cap = L.ring;
      G.ring_first = gbase + R0;
      G.base = a;
      G.end = end;
      vmps_stats_t cs;
      const double t0 = bd_now(s);
      r2 = sort_impl<KT, HV>(w, (char*)keys + a * kb, HV ? vals + a : nullptr, s, st ? &cs : nullptr, &G);
      bd_add(5, t0, s);
      if (r2 != VMPS_OK) return r2;
      if (st) {
        M += cs.merge_cost_M;
        maxp = std::max(maxp, cs.max_power);
        lv = std::max(lv, cs.levels_executed);
      }
    }
    runs += m;
    if (st) {
      for (size_t i = 0; i < m; ++i) {
        if (RKr[i] & 1u) rev += (i + 1 < m ? Rr[i + 1] : end) - Rr[i];
        if (RKr[i] & 2u) ++ext;
      }
    }
    const Seg nx{a, end, m > 1 ? Rr[1] : end, Rr[m - 1], 0};
    R0 += m;
    if (R0 > (1u << 16) && R0 * 2 > R.size()) {  // drop the consumed prefix
      R.erase(R.begin(), R.begin() + R0);
      RK.erase(RK.begin(), RK.begin() + R0);
      gbase += R0;
      R0 = 0;
    }
    return push_cell(nx);
  };
  // Close every cell whose last run's end is known: runs R[R0, R0+m) share a
  // cell and run R0+m (whose start is the end of run R0+m-1) lies in a later one.
  auto close_cells = [&]() -> vmps_status_t {
    for (;;) {
      const double tc = bd_now(s);
      const size_t avail = R.size() - R0;
      if (avail < 2) break;
      const uint64_t* Rr = R.data() + R0;
      const uint64_t T = cell_end(cell_of(Rr[0], Rr[1]));
      size_t m = 1;
      while (m + 1 < avail && Rr[m] + Rr[m + 1] < T) ++m;
      if (m + 1 >= avail) break;  // run m's end unknown or run m still in the cell
      bd_add(8, tc, s);
      vmps_status_t r2 = do_cell(m, Rr[m]);
      if (r2 != VMPS_OK) return r2;
    }
    return VMPS_OK;
  };
  // Scan: detection chunk by chunk on a second stream, one chunk ahead of the
  // cells.  While the cells closed by the runs of chunks < i run on s, the
  // runs of chunk i and the chain table of chunk i+1 are computed on sd.  No
  // cell reaches chunk i: a closed cell ends at a known run start (< the start
  // of chunk i, a block boundary), so chunk i's blocks, its halo and its last
  // key are still the caller's originals when sd reads them.  The ring copy of
  // chunk i's runs waits for the cells issued one iteration earlier (the ring
  // holds an open cell's runs and two chunks').
  if (!g_det_host.reserve(ns, rdet)) { g_err = "cudaMallocHost (detection staging)"; return VMPS_ERR_CUDA; }
  DetHost& hb = g_det_host;
  struct StreamGuard {
    cudaStream_t sd = nullptr;
    cudaEvent_t ev = nullptr;
    ~StreamGuard() {
      if (sd) { cudaStreamSynchronize(sd); cudaStreamDestroy(sd); }
      if (ev) cudaEventDestroy(ev);
    }
  } sg;
  VMPS_CK(cudaStreamCreateWithFlags(&sg.sd, cudaStreamNonBlocking));
  VMPS_CK(cudaEventCreateWithFlags(&sg.ev, cudaEventDisableTiming));
  cudaStream_t sd = sg.sd;
  uint32_t state = 0;  // START(0)
  if (bd_trace()) memset(&g_bdt, 0, sizeof(g_bdt));
  const double t_all = bd_now(s);
  const uint64_t nchunks = (n + L.det - 1) / L.det;
  struct ChunkArgs { uint64_t off, nd; uint32_t n_halo, n_end; const K* kk; };
  auto chunk = [&](uint64_t i) -> ChunkArgs {
    ChunkArgs c;
    c.off = i * L.det;
    c.nd = std::min<uint64_t>(L.det, n - c.off);
    c.n_halo = (uint32_t)std::min<uint64_t>(H, n - c.off - c.nd);
    const uint64_t rem = n - c.off;
    c.n_end = rem >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)rem;
    c.kk = (const K*)((const char*)keys + c.off * kb);
    return c;
  };
  auto issue_chain = [&](uint64_t i) -> vmps_status_t {
    const ChunkArgs c = chunk(i);
    vmps_status_t r2 = vmps_shard_chain(c.kk, c.nd, (vmps_key_t)KT, minrun, c.n_end, c.off ? d_prev : nullptr,
                                        c.n_halo ? (const void*)(c.kk + c.nd) : nullptr, c.n_halo, d_tab, det_ws,
                                        L.det_ws, sd);
    if (r2 != VMPS_OK) return r2;
    VMPS_CK(cudaMemcpyAsync(hb.tab, d_tab, (size_t)ns * 8, cudaMemcpyDeviceToHost, sd));
    return VMPS_OK;
  };
  rc = issue_chain(0);
  if (rc != VMPS_OK) return rc;
  uint32_t pending = 0;  // runs of the previous chunk staged in hb.rs / hb.rk
  for (uint64_t i = 0; i < nchunks; ++i) {
    const double t_det = bd_now(s);
    VMPS_CK(cudaStreamSynchronize(sd));
    if (pending) {  // runs of chunk i-1: to the host list (their ring copy is complete)
      const size_t o = R.size();
      R.insert(R.end(), hb.rs, hb.rs + pending);
      RK.insert(RK.end(), hb.rk, hb.rk + pending);
      (void)o;
      pending = 0;
    }
    const ChunkArgs c = chunk(i);
    const uint64_t v = hb.tab[state];
    const uint32_t cnt = (uint32_t)(v & 0xFFFFFFFFull);
    if (cnt) {
      rc = shard_runs_impl(c.kk, c.nd, (vmps_key_t)KT, minrun, c.n_end, c.off ? d_prev : nullptr,
                           c.n_halo ? (const void*)(c.kk + c.nd) : nullptr, c.n_halo, state, cnt, c.off, d_rs, d_rk,
                           det_ws, L.det_ws, sd, true);
      if (rc != VMPS_OK) return rc;
      VMPS_CK(cudaMemcpyAsync(hb.rs, d_rs, (size_t)cnt * 8, cudaMemcpyDeviceToHost, sd));
      VMPS_CK(cudaMemcpyAsync(hb.rk, d_rk, cnt, cudaMemcpyDeviceToHost, sd));
    }
    state = (uint32_t)(v >> 32);
    // the original last key of this chunk (the next chunk's descent bit at its start)
    VMPS_CK(cudaMemcpyAsync(d_prev, c.kk + c.nd - 1, kb, cudaMemcpyDeviceToDevice, sd));
    if (i + 1 < nchunks) {
      rc = issue_chain(i + 1);
      if (rc != VMPS_OK) return rc;
    }
    if (cnt) {  // into the device ring the cells read their runs from
      if (R.size() - R0 + cnt > L.ring) { g_err = "internal: run ring"; return VMPS_ERR_INTERNAL; }
      VMPS_CK(cudaStreamWaitEvent(sd, sg.ev, 0));  // the cells of the previous iteration are done
      const uint64_t at = g_total % L.ring, n1 = std::min<uint64_t>(cnt, L.ring - at);
      VMPS_CK(cudaMemcpyAsync(d_ring + at, d_rs, n1 * 8, cudaMemcpyDeviceToDevice, sd));
      VMPS_CK(cudaMemcpyAsync(d_ring_kind + at, d_rk, n1, cudaMemcpyDeviceToDevice, sd));
      if (n1 < cnt) {
        VMPS_CK(cudaMemcpyAsync(d_ring, d_rs + n1, (cnt - n1) * 8, cudaMemcpyDeviceToDevice, sd));
        VMPS_CK(cudaMemcpyAsync(d_ring_kind, d_rk + n1, cnt - n1, cudaMemcpyDeviceToDevice, sd));
      }
      g_total += cnt;
      pending = cnt;
    }
    bd_add(4, t_det, s);
    rc = close_cells();
    if (rc != VMPS_OK) return rc;
    VMPS_CK(cudaEventRecord(sg.ev, s));  // the next ring copy waits for these cells
  }
  VMPS_CK(cudaStreamSynchronize(sd));
  if (pending) {
    R.insert(R.end(), hb.rs, hb.rs + pending);
    RK.insert(RK.end(), hb.rk, hb.rk + pending);
    pending = 0;
  }
  rc = close_cells();
  if (rc != VMPS_OK) return rc;
  // the array is done: remaining runs end at n
  while (R0 < R.size()) {
    const size_t avail = R.size() - R0;
    const uint64_t* Rr = R.data() + R0;
    const auto end_of = [&](size_t i) { return i + 1 < avail ? Rr[i + 1] : n; };
    const uint64_t T = cell_end(cell_of(Rr[0], end_of(0)));
    size_t m = 1;
    while (m < avail && Rr[m] + end_of(m) < T) ++m;
    rc = do_cell(m, m < avail ? Rr[m] : n);
    if (rc != VMPS_OK) return rc;
  }
  // lines 12-13: pop and merge what is left
  while (!stk.empty()) {
    rc = merge2(stk.back(), curr);
    if (rc != VMPS_OK) return rc;
    curr = Seg{stk.back().a, curr.b, stk.back().first_end, curr.last_start, 0};
    stk.pop_back();
  }
  rc = bd_check(C, s, "mode");
  if (rc != VMPS_OK) return rc;
  // one Copy for the whole array
  const double t_cp = bd_now(s);
  rc = bd_copy<KT, HV>(C, s);
  if (rc == VMPS_OK) rc = bd_check(C, s, "Copy");
  if (rc != VMPS_OK) return rc;
  bd_add(2, t_cp, s);
  if (bd_trace()) {
    bd_add(7, t_all, s);
    static const char* nm[10] = {"home", "levels", "copy", "front+leaf", "detect", "cell_sorts", "top_merges", "all",
                                 "close", "do_cell"};
    for (int i = 0; i < 10; ++i) fprintf(stderr, "vmps bd trace: %-10s %9.1f ms  %ld\n", nm[i], g_bdt.t[i], g_bdt.n[i]);
  }
  if (st) {
    BdState hs;
    VMPS_CK(cudaMemcpyAsync(&hs, C.bstate, sizeof(hs), cudaMemcpyDeviceToHost, s));
    VMPS_CK(cudaStreamSynchronize(s));
    memset(st, 0, sizeof(*st));
    st->n = n;
    st->runs = runs;
    st->merges = runs ? runs - 1 : 0;
    st->merge_cost_M = M;
    st->reversed_elems = rev;
    st->extended_runs = ext;
    st->max_power = maxp;
    st->levels_executed = lv;
    st->minrun = minrun;
    st->block_elems = c0.P;
    st->rounds = hs.rounds;
    st->scratch_bytes = (uint64_t)c0.F * c0.P * (kb + (HV ? 4 : 0));
    st->peak_extra_device_bytes = L.total;
    st->metadata_bytes = L.total - st->scratch_bytes;
  }
  return VMPS_OK;
}

static vmps_status_t merge_runs_bounded_impl(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt,
                                             const uint64_t* h_run_start, uint32_t nruns, int64_t scratch_elems,
                                             void* ws, size_t ws_bytes, void* stream);

extern "C" {

static vmps_status_t sort_any(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt, int64_t scratch_elems,
                              void* ws, size_t ws_bytes, void* stream, vmps_stats_t* h_stats) {
  vmps_status_t rc = check_common(keys, vals, n, kt);
  if (rc != VMPS_OK) return rc;
  if (scratch_elems != VMPS_SCRATCH_UNBOUNDED && scratch_elems < 0) {
    g_err = "scratch_elems must be >= 0 or VMPS_SCRATCH_UNBOUNDED";
    return VMPS_ERR_INVALID_ARG;
  }
  if (n <= 1) {
    if (h_stats) { memset(h_stats, 0, sizeof(*h_stats)); h_stats->n = n; h_stats->runs = n; }
    return VMPS_OK;
  }
  const int hv = vals ? 1 : 0;
  Cfg c = make_cfg(n, kt, hv, scratch_elems);
  if (scratch_elems >= 0 && c.F < BD_MIN_BLOCKS) {
    g_err = "scratch_elems below the bounded mode's minimum (6 blocks)";
    return VMPS_ERR_BUDGET;
  }
  if (bd_chunked(n, scratch_elems, hv)) {
    const size_t need = bd_cell_layout(n, kt, hv, scratch_elems).total;
    char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    if (!ws || ws_bytes < need || (size_t)(base - (char*)ws) + need > ws_bytes) {
      g_err = "workspace too small";
      return VMPS_ERR_BUDGET;
    }
    cudaStream_t s = (cudaStream_t)stream;
    switch (kt) {
      case VMPS_KEY_U32:
        return hv ? sort_bounded_cells<VMPS_KEY_U32, true>(keys, vals, n, scratch_elems, base, s, h_stats)
                  : sort_bounded_cells<VMPS_KEY_U32, false>(keys, vals, n, scratch_elems, base, s, h_stats);
      case VMPS_KEY_U64:
        return hv ? sort_bounded_cells<VMPS_KEY_U64, true>(keys, vals, n, scratch_elems, base, s, h_stats)
                  : sort_bounded_cells<VMPS_KEY_U64, false>(keys, vals, n, scratch_elems, base, s, h_stats);
      default:
        return hv ? sort_bounded_cells<VMPS_KEY_F32, true>(keys, vals, n, scratch_elems, base, s, h_stats)
                  : sort_bounded_cells<VMPS_KEY_F32, false>(keys, vals, n, scratch_elems, base, s, h_stats);
    }
  }
  Work w;
  size_t need = carve(c, &w, nullptr);
  if (!ws || ws_bytes < need) {
    g_err = "workspace too small";
    return VMPS_ERR_BUDGET;
  }
  char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if ((size_t)(base - (char*)ws) + need > ws_bytes) {
    g_err = "workspace too small after alignment";
    return VMPS_ERR_BUDGET;
  }
  carve(c, &w, base);
  cudaStream_t s = (cudaStream_t)stream;
  switch (kt) {
    case VMPS_KEY_U32:
      return hv ? sort_impl<VMPS_KEY_U32, true>(w, keys, vals, s, h_stats)
                : sort_impl<VMPS_KEY_U32, false>(w, keys, vals, s, h_stats);
    case VMPS_KEY_U64:
      return hv ? sort_impl<VMPS_KEY_U64, true>(w, keys, vals, s, h_stats)
                : sort_impl<VMPS_KEY_U64, false>(w, keys, vals, s, h_stats);
    default:
      return hv ? sort_impl<VMPS_KEY_F32, true>(w, keys, vals, s, h_stats)
                : sort_impl<VMPS_KEY_F32, false>(w, keys, vals, s, h_stats);
  }
}

vmps_status_t vmps_sort_keys(void* keys, uint64_t n, vmps_key_t kt, int64_t scratch_elems, void* ws,
                             size_t ws_bytes, void* stream, vmps_stats_t* h_stats) {
  return sort_any(keys, nullptr, n, kt, scratch_elems, ws, ws_bytes, stream, h_stats);
}

vmps_status_t vmps_sort_pairs(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt, int64_t scratch_elems,
                              void* ws, size_t ws_bytes, void* stream, vmps_stats_t* h_stats) {
  if (n > 1 && !vals) {
    g_err = "vals is NULL";
    return VMPS_ERR_INVALID_ARG;
  }
  return sort_any(keys, vals, n, kt, scratch_elems, ws, ws_bytes, stream, h_stats);
}

static vmps_status_t sort_host_any(const void* h_keys, const uint32_t* h_vals, void* h_kout, uint32_t* h_vout,
                                   uint64_t n, vmps_key_t kt, int64_t scratch_elems, void* d_keys,
                                   uint32_t* d_vals, void* ws, size_t ws_bytes, void* stream,
                                   vmps_stats_t* h_stats, bool pairs) {
  if (n > 1 && (!h_keys || !d_keys || (pairs && (!h_vals || !d_vals)))) {
    g_err = "host or device buffer is NULL";
    return VMPS_ERR_INVALID_ARG;
  }
  vmps_status_t rc = check_common(d_keys, pairs ? d_vals : nullptr, n, kt);
  if (rc != VMPS_OK) return rc;
  if (n <= 1) {  // nothing to sort; an out-of-place call still copies the item
    if (n == 1 && h_kout) memcpy(h_kout, h_keys, key_bytes(kt));
    if (n == 1 && pairs && h_vout) memcpy(h_vout, h_vals, 4);
    if (h_stats) { memset(h_stats, 0, sizeof(*h_stats)); h_stats->n = n; h_stats->runs = n; }
    return VMPS_OK;
  }
  // validate the budget before anything is enqueued
  if (scratch_elems != VMPS_SCRATCH_UNBOUNDED && scratch_elems < 0) {
    g_err = "scratch_elems must be >= 0 or VMPS_SCRATCH_UNBOUNDED";
    return VMPS_ERR_INVALID_ARG;
  }
  if (scratch_elems >= 0 && make_cfg(n, kt, pairs ? 1 : 0, scratch_elems).F < BD_MIN_BLOCKS) {
    g_err = "scratch_elems below the bounded mode's minimum (6 blocks)";
    return VMPS_ERR_BUDGET;
  }
  size_t need = 0;
  vmps_workspace_bytes(n, kt, pairs ? 1 : 0, scratch_elems, &need);
  if (!ws || ws_bytes < need) { g_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t kb = (size_t)n * key_bytes(kt), vb = (size_t)n * 4;
  VMPS_CK(cudaMemcpyAsync(d_keys, h_keys, kb, cudaMemcpyHostToDevice, s));
  if (pairs) VMPS_CK(cudaMemcpyAsync(d_vals, h_vals, vb, cudaMemcpyHostToDevice, s));
  // stats (if requested) synchronise inside the sort; read-back follows
  rc = sort_any(d_keys, pairs ? d_vals : nullptr, n, kt, scratch_elems, ws, ws_bytes, stream, nullptr);
  if (rc != VMPS_OK) return rc;
  void* ko = h_kout ? h_kout : const_cast<void*>(h_keys);
  uint32_t* vo = h_vout ? h_vout : const_cast<uint32_t*>(h_vals);
  VMPS_CK(cudaMemcpyAsync(ko, d_keys, kb, cudaMemcpyDeviceToHost, s));
  if (pairs) VMPS_CK(cudaMemcpyAsync(vo, d_vals, vb, cudaMemcpyDeviceToHost, s));
  if (h_stats) {
    VMPS_CK(cudaStreamSynchronize(s));
    memset(h_stats, 0, sizeof(*h_stats));
    h_stats->n = n;
  }
  return VMPS_OK;
}

vmps_status_t vmps_sort_keys_host(const void* h_keys, void* h_keys_out, uint64_t n, vmps_key_t kt,
                                  int64_t scratch_elems, void* d_keys, void* ws, size_t ws_bytes, void* stream,
                                  vmps_stats_t* h_stats) {
  return sort_host_any(h_keys, nullptr, h_keys_out, nullptr, n, kt, scratch_elems, d_keys, nullptr, ws, ws_bytes,
                       stream, h_stats, false);
}

vmps_status_t vmps_sort_pairs_host(const void* h_keys, const uint32_t* h_vals, void* h_keys_out,
                                   uint32_t* h_vals_out, uint64_t n, vmps_key_t kt, int64_t scratch_elems,
                                   void* d_keys, uint32_t* d_vals, void* ws, size_t ws_bytes, void* stream,
                                   vmps_stats_t* h_stats) {
  return sort_host_any(h_keys, h_vals, h_keys_out, h_vals_out, n, kt, scratch_elems, d_keys, d_vals, ws, ws_bytes,
                       stream, h_stats, true);
}

vmps_status_t vmps_merge_plan(const void* keys, uint64_t n, vmps_key_t kt, uint64_t* run_start,
                              uint8_t* run_kind, vmps_merge_rec_t* merges, uint64_t cap_runs,
                              uint64_t* h_num_runs, void* ws, size_t ws_bytes, void* stream) {
  vmps_status_t rc = check_common(keys, nullptr, n, kt);
  if (rc != VMPS_OK) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 1) {
    if (h_num_runs) *h_num_runs = n;
    if (n == 1) {
      if (cap_runs < 1 || !run_start || !run_kind) { g_err = "cap_runs too small"; return VMPS_ERR_INVALID_ARG; }
      uint64_t z = 0;
      uint8_t kz = 0;
      VMPS_CK(cudaMemcpyAsync(run_start, &z, 8, cudaMemcpyHostToDevice, s));
      VMPS_CK(cudaMemcpyAsync(run_kind, &kz, 1, cudaMemcpyHostToDevice, s));
      VMPS_CK(cudaStreamSynchronize(s));
    }
    return VMPS_OK;
  }
  if (!run_start || !run_kind || !merges) { g_err = "plan output is NULL"; return VMPS_ERR_INVALID_ARG; }
  Cfg c = make_cfg(n, kt, -1);
  Work w;
  size_t need = carve(c, &w, nullptr);
  if (!ws || ws_bytes < need) { g_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if ((size_t)(base - (char*)ws) + need > ws_bytes) { g_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  carve(c, &w, base);
  switch (kt) {
    case VMPS_KEY_U32: rc = front_half<VMPS_KEY_U32>(w, keys, s); break;
    case VMPS_KEY_U64: rc = front_half<VMPS_KEY_U64>(w, keys, s); break;
    default: rc = front_half<VMPS_KEY_F32>(w, keys, s); break;
  }
  if (rc != VMPS_OK) return rc;
  uint32_t r = 0;
  VMPS_CK(cudaMemcpyAsync(&r, w.scalars + SC_RUNS, 4, cudaMemcpyDeviceToHost, s));
  VMPS_CK(cudaStreamSynchronize(s));
  if (h_num_runs) *h_num_runs = r;
  if (r > cap_runs) { g_err = "cap_runs too small"; return VMPS_ERR_INVALID_ARG; }
  k_plan_records<uint32_t><<<grid_for(r), 256, 0, s>>>(w.run_start, w.scalars, w.power, w.seg_l, w.seg_r, w.dep[0],
                                             w.run_kind, run_start, run_kind, merges);
  rc = launch_check();
  if (rc != VMPS_OK) return rc;
  VMPS_CK(cudaStreamSynchronize(s));
  return VMPS_OK;
}

static bool shard_args_ok(const void* keys, uint64_t n_local, vmps_key_t kt, uint32_t minrun, uint32_t n_halo) {
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) { g_err = "unknown key type"; return false; }
  if (n_local < 1 || n_local > VMPS_MAX_N || !keys) {
    g_err = "shard: need 1 <= n_local <= VMPS_MAX_N keys";
    return false;
  }
  if (minrun < 1 || minrun > MAX_MINRUN) { g_err = "shard: minrun out of range"; return false; }
  if (n_halo > 2 * MAX_MINRUN + 8) { g_err = "shard: halo too long"; return false; }
  if ((uintptr_t)keys & 15) { g_err = "keys must be 16-byte aligned"; return false; }
  return true;
}

static Cfg shard_cfg(uint64_t n_local, vmps_key_t kt, uint32_t minrun) {
  Cfg c = make_cfg(n_local, kt, -1);
  c.minrun = minrun;
  return c;
}

vmps_status_t vmps_shard_workspace_bytes(uint64_t n_local, vmps_key_t kt, uint32_t minrun, size_t* h_bytes) {
  if (!h_bytes || n_local < 1 || n_local > VMPS_MAX_N || minrun < 1 || minrun > MAX_MINRUN)
    return VMPS_ERR_INVALID_ARG;
  *h_bytes = carve(shard_cfg(n_local, kt, minrun), nullptr, nullptr) + 256;
  return VMPS_OK;
}

static vmps_status_t shard_setup(const void* keys, uint64_t n_local, vmps_key_t kt, uint32_t minrun,
                                 uint32_t n_end, uint32_t n_halo, void* ws, size_t ws_bytes, Work* w) {
  if (!shard_args_ok(keys, n_local, kt, minrun, n_halo)) return VMPS_ERR_INVALID_ARG;
  if (n_end < n_local) { g_err = "shard: n_end < n_local"; return VMPS_ERR_INVALID_ARG; }
  const Cfg c = shard_cfg(n_local, kt, minrun);
  const size_t need = carve(c, nullptr, nullptr);
  char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if (!ws || (size_t)(base - (char*)ws) + need > ws_bytes) { g_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  carve(c, w, base);
  return VMPS_OK;
}

vmps_status_t vmps_shard_chain(const void* keys, uint64_t n_local, vmps_key_t kt, uint32_t minrun, uint32_t n_end,
                               const void* d_prev, const void* d_halo, uint32_t n_halo, uint64_t* d_table,
                               void* ws, size_t ws_bytes, void* stream) {
  Work w;
  vmps_status_t rc = shard_setup(keys, n_local, kt, minrun, n_end, n_halo, ws, ws_bytes, &w);
  if (rc != VMPS_OK) return rc;
  if (!d_table) { g_err = "table output is NULL"; return VMPS_ERR_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  switch (kt) {
    case VMPS_KEY_U32: rc = shard_dispatch_front<VMPS_KEY_U32>(w, keys, n_end, d_prev, d_halo, n_halo, s); break;
    case VMPS_KEY_U64: rc = shard_dispatch_front<VMPS_KEY_U64>(w, keys, n_end, d_prev, d_halo, n_halo, s); break;
    default: rc = shard_dispatch_front<VMPS_KEY_F32>(w, keys, n_end, d_prev, d_halo, n_halo, s); break;
  }
  if (rc != VMPS_OK) return rc;
  const int top = w.chain_levels;
  if (top == 0) k_chain_all<uint32_t><<<1, 256, 0, s>>>(w.tile_tab, w.chain_m[0], w.ns, d_table);
  else k_chain_all<uint64_t><<<1, 256, 0, s>>>(w.chain_tab[top - 1], w.chain_m[top], w.ns, d_table);
  return launch_check();
}

}  // extern "C"
// front_done: the workspace already holds this shard's tables (the previous
// call on it was vmps_shard_chain with the same arguments, same stream)
static vmps_status_t shard_runs_impl(const void* keys, uint64_t n_local, vmps_key_t kt, uint32_t minrun,
                                     uint32_t n_end, const void* d_prev, const void* d_halo, uint32_t n_halo,
                                     uint32_t entry_state, uint64_t count, uint64_t offset, uint64_t* d_run_start,
                                     uint8_t* d_run_kind, void* ws, size_t ws_bytes, void* stream, bool front_done) {
  Work w;
  vmps_status_t rc = shard_setup(keys, n_local, kt, minrun, n_end, n_halo, ws, ws_bytes, &w);
  if (rc != VMPS_OK) return rc;
  if (entry_state > ST_END || (entry_state != ST_END && entry_state >= 3 * minrun)) {
    g_err = "shard: bad entry state";
    return VMPS_ERR_INVALID_ARG;
  }
  if (count > w.rmax || (count && (!d_run_start || !d_run_kind))) { g_err = "shard: bad run count"; return VMPS_ERR_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  if (!front_done) {
    switch (kt) {
      case VMPS_KEY_U32: rc = shard_dispatch_front<VMPS_KEY_U32>(w, keys, n_end, d_prev, d_halo, n_halo, s); break;
      case VMPS_KEY_U64: rc = shard_dispatch_front<VMPS_KEY_U64>(w, keys, n_end, d_prev, d_halo, n_halo, s); break;
      default: rc = shard_dispatch_front<VMPS_KEY_F32>(w, keys, n_end, d_prev, d_halo, n_halo, s); break;
    }
    if (rc != VMPS_OK) return rc;
  }
  const int top = w.chain_levels;
  const size_t sm32 = (size_t)CHAIN_G * w.ns * 4, sm64 = (size_t)CHAIN_G * w.ns * 8;
  if (top == 0)
    LAUNCH(k_chain_top<uint32_t>, 1, 32, 0, s, w.tile_tab, w.chain_m[0], w.ns, w.chain_entry[0], entry_state);
  else
    LAUNCH(k_chain_top<uint64_t>, 1, 32, 0, s, w.chain_tab[top - 1], w.chain_m[top], w.ns, w.chain_entry[top],
           entry_state);
  for (int l = top - 1; l >= 0; --l) {
    if (l == 0)
      LAUNCH(k_chain_expand<uint32_t>, w.chain_m[1], 256, sm32, s, w.tile_tab, w.chain_m[0], w.ns,
             w.chain_entry[1], w.chain_entry[0]);
    else
      LAUNCH(k_chain_expand<uint64_t>, w.chain_m[l + 1], 256, sm64, s, w.chain_tab[l - 1], w.chain_m[l], w.ns,
             w.chain_entry[l + 1], w.chain_entry[l]);
  }
  LAUNCH(k_runs_emit, w.ntiles, 128, 0, s, w.bits, w.n, w.minrun, w.chain_entry[0], w.run_start, w.run_kind,
         w.scalars, n_end, n_halo);
  if (count) {
    LAUNCH(k_shard_starts, grid_for(count), 256, 0, s, w.run_start, count, offset, d_run_start);
    VMPS_CK(cudaMemcpyAsync(d_run_kind, w.run_kind, count, cudaMemcpyDeviceToDevice, s));
  }
  return launch_check();
}
extern "C" {
vmps_status_t vmps_shard_runs(const void* keys, uint64_t n_local, vmps_key_t kt, uint32_t minrun, uint32_t n_end,
                              const void* d_prev, const void* d_halo, uint32_t n_halo, uint32_t entry_state,
                              uint64_t count, uint64_t offset, uint64_t* d_run_start, uint8_t* d_run_kind, void* ws,
                              size_t ws_bytes, void* stream) {
  return shard_runs_impl(keys, n_local, kt, minrun, n_end, d_prev, d_halo, n_halo, entry_state, count, offset,
                         d_run_start, d_run_kind, ws, ws_bytes, stream, false);
}

// The merge plan of an array given its run starts (64-bit positions, r + 1
// entries with run_start[r] = n): powers, tree, Alg. 1 order -- the back half
// of vmps_merge_plan, for run lists assembled from shards (n may exceed 2^32).
vmps_status_t vmps_plan_workspace_bytes(uint64_t r, size_t* h_bytes) {
  if (!h_bytes || r >= (1ull << 32) - 8) return VMPS_ERR_INVALID_ARG;
  const size_t R = (size_t)r + 2;
  *h_bytes = 256 * 10 + R * (1 + 4 * 7) + SC_COUNT * 4 + 64;
  return VMPS_OK;
}

vmps_status_t vmps_plan_from_runs(const uint64_t* d_run_start, uint64_t r, uint64_t n, vmps_merge_rec_t* d_merges,
                                  void* ws, size_t ws_bytes, void* stream) {
  size_t need = 0;
  if (vmps_plan_workspace_bytes(r, &need) != VMPS_OK || r < 1 || n < r || !d_run_start) {
    g_err = "plan_from_runs: bad arguments";
    return VMPS_ERR_INVALID_ARG;
  }
  if (r >= 2 && !d_merges) { g_err = "plan_from_runs: merges is NULL"; return VMPS_ERR_INVALID_ARG; }
  if (!ws || ws_bytes < need) { g_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  if (r < 2) return VMPS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  size_t off = 0;
  auto take = [&](size_t bytes) { void* p = base + off; off += (bytes + 255) & ~(size_t)255; return p; };
  const size_t R = (size_t)r + 2;
  uint8_t* power = (uint8_t*)take(R);
  uint32_t* seg_l = (uint32_t*)take(R * 4);
  uint32_t* seg_r = (uint32_t*)take(R * 4);
  uint32_t* parent = (uint32_t*)take(R * 4);
  uint32_t* anc0 = (uint32_t*)take(R * 4);
  uint32_t* anc1 = (uint32_t*)take(R * 4);
  uint32_t* dep0 = (uint32_t*)take(R * 4);
  uint32_t* dep1 = (uint32_t*)take(R * 4);
  uint32_t* scal = (uint32_t*)take(SC_COUNT * 4 + 64);
  uint32_t hs[SC_COUNT] = {0};
  hs[SC_RUNS] = (uint32_t)r;
  VMPS_CK(cudaMemcpyAsync(scal, hs, sizeof(hs), cudaMemcpyHostToDevice, s));
  const unsigned g = grid_for(r);
  LAUNCH(k_powers_seg<uint64_t>, g, 256, 0, s, d_run_start, n, scal, power, seg_l, seg_r);
  LAUNCH(k_parent_init, g, 256, 0, s, scal, power, seg_l, seg_r, parent, anc0, dep0);
  uint32_t *anc[2] = {anc0, anc1}, *dep[2] = {dep0, dep1};
  for (int rnd = 0; rnd < 6; ++rnd) {
    int a = rnd & 1;
    LAUNCH(k_jump, g, 256, 0, s, scal, anc[a], dep[a], anc[a ^ 1], dep[a ^ 1]);
  }
  // records only (run starts / kinds are the caller's)
  k_plan_records_only<<<g, 256, 0, s>>>(d_run_start, scal, power, seg_l, seg_r, dep0, d_merges);
  VMPS_CK(cudaStreamSynchronize(s));  // the host array hs must outlive the copy
  return launch_check();
}

const char* vmps_status_string(vmps_status_t s) {
  switch (s) {
    case VMPS_OK: return "ok";
    case VMPS_ERR_INVALID_ARG: return "invalid argument";
    case VMPS_ERR_ALLOC: return "allocation failed";
    case VMPS_ERR_BUDGET: return "workspace or scratch budget too small";
    case VMPS_ERR_CUDA: return "CUDA error";
    case VMPS_ERR_NCCL: return "NCCL error";
    case VMPS_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

const char* vmps_last_error(void) { return g_err.c_str(); }

void vmps_profile_enable(int on) { g_prof = on != 0; }

int vmps_profile_read(double* h_ms, int cap, uint64_t* h_launches, uint64_t* h_bytes) {
  if (h_launches) { h_launches[0] = g_nl; h_launches[1] = g_nl_merge; }
  if (!g_prof || g_prof_mark[0] < 0 || g_prof_mark[3] < 0) return 0;
  auto el = [](int a, int b) -> double {
    float ms = 0.f;
    if (a < 0 || b < 0) return 0.0;
    if (cudaEventElapsedTime(&ms, g_ev[a], g_ev[b]) != cudaSuccess) return -1.0;
    return (double)ms;
  };
  double v[5];
  v[0] = el(g_prof_mark[0], g_prof_mark[1]);
  v[1] = el(g_prof_mark[1], g_prof_mark[2]);
  v[2] = 0.0;
  for (int i = 0; i < g_prof_np; ++i) v[2] += el(g_prof_part[i][0], g_prof_part[i][1]);
  v[3] = 0.0;
  for (int i = 0; i < g_prof_nm; ++i) v[3] += el(g_prof_lvl[i][0], g_prof_lvl[i][1]);
  v[4] = el(g_prof_mark[0], g_prof_mark[3]);
  int k = 0;
  for (; k < cap && k < 5; ++k) h_ms[k] = v[k];
  if (h_bytes && g_prof_host) {
    unsigned long long M = g_prof_host[0], fM = g_prof_host[1], hM = g_prof_host[2];
    h_bytes[0] = 2ull * (unsigned long long)g_prof_wbytes * hM;  // read + write of every HBM merge
    h_bytes[1] = M;
    h_bytes[2] = fM;
  }
  return k;
}

void vmps_test_set_mode(int levels_per_pass) { g_fuse2 = levels_per_pass == 1 ? 0 : 1; }

void vmps_test_set_leaf(int radix) { g_leaf_radix = radix ? 1 : 0; }

// ---- scratch-bounded merge of given sorted runs (the multi-GPU bounded
// protocol's re-merge after a swap; csrc/comm.cu) ----
vmps_status_t vmps_merge_runs_bounded_workspace_bytes(uint64_t n, vmps_key_t kt, int has_vals, uint32_t nruns,
                                                      int64_t scratch_elems, size_t* h_bytes) {
  if (!h_bytes || n > VMPS_MAX_N || nruns < 1 || scratch_elems < 0) return VMPS_ERR_INVALID_ARG;
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) return VMPS_ERR_INVALID_ARG;
  if (n <= 1) { *h_bytes = 256; return VMPS_OK; }
  Cfg c = make_cfg(n, kt, has_vals ? 1 : 0, scratch_elems);
  c.given_runs = nruns;
  *h_bytes = carve(c, nullptr, nullptr) + 256;
  return VMPS_OK;
}

vmps_status_t vmps_merge_runs_bounded(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt,
                                      const uint64_t* h_run_start, uint32_t nruns, int64_t scratch_elems, void* ws,
                                      size_t ws_bytes, void* stream) {
  vmps_status_t rc = check_common(keys, vals, n, kt);
  if (rc != VMPS_OK) return rc;
  return merge_runs_bounded_impl(keys, vals, n, kt, h_run_start, nruns, scratch_elems, ws, ws_bytes, stream);
}

}  // extern "C"

// (no alignment requirement: the bounded engine's kernels access elements
// one by one, so sub-arrays at any element offset are fine)
static vmps_status_t merge_runs_bounded_impl(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt,
                                             const uint64_t* h_run_start, uint32_t nruns, int64_t scratch_elems,
                                             void* ws, size_t ws_bytes, void* stream) {
  if (scratch_elems < 0 || !h_run_start || nruns < 1) { g_err = "bad arguments"; return VMPS_ERR_INVALID_ARG; }
  if (n <= 1) return VMPS_OK;
  // distinct starts inside [0, n), ascending from 0
  std::vector<uint32_t> runs;
  for (uint32_t q = 0; q < nruns; ++q) {
    const uint64_t a = h_run_start[q];
    if (a >= n || (q && a <= h_run_start[q - 1])) continue;
    if (runs.empty() && a != 0) runs.push_back(0);
    runs.push_back((uint32_t)a);
  }
  if (runs.empty() || runs[0] != 0) runs.insert(runs.begin(), 0u);
  if (runs.size() < 2) return VMPS_OK;  // one run: already sorted
  const uint32_t r = (uint32_t)runs.size();
  runs.push_back((uint32_t)n);
  const int hv = vals ? 1 : 0;
  Cfg c = make_cfg(n, kt, hv, scratch_elems);
  if (c.F < BD_MIN_BLOCKS) { g_err = "scratch_elems below the bounded mode's minimum (6 blocks)"; return VMPS_ERR_BUDGET; }
  c.given_runs = r;
  Work w;
  const size_t need = carve(c, &w, nullptr);
  char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if (!ws || ws_bytes < need || (size_t)(base - (char*)ws) + need > ws_bytes) {
    g_err = "workspace too small";
    return VMPS_ERR_BUDGET;
  }
  carve(c, &w, base);
  cudaStream_t s = (cudaStream_t)stream;
  const GivenRuns G{runs.data(), nullptr, nullptr, n, r};
  switch (kt) {
    case VMPS_KEY_U32:
      return hv ? sort_impl<VMPS_KEY_U32, true>(w, keys, vals, s, nullptr, &G)
                : sort_impl<VMPS_KEY_U32, false>(w, keys, vals, s, nullptr, &G);
    case VMPS_KEY_U64:
      return hv ? sort_impl<VMPS_KEY_U64, true>(w, keys, vals, s, nullptr, &G)
                : sort_impl<VMPS_KEY_U64, false>(w, keys, vals, s, nullptr, &G);
    default:
      return hv ? sort_impl<VMPS_KEY_F32, true>(w, keys, vals, s, nullptr, &G)
                : sort_impl<VMPS_KEY_F32, false>(w, keys, vals, s, nullptr, &G);
  }
}

extern "C" {

void vmps_test_set_bd_chunk(uint32_t chunk) { g_bd_chunk = chunk ? std::max<uint32_t>(chunk, 4096u) : VMPS_BD_CHUNK; }

void vmps_test_set_minrun(uint32_t minrun) { g_minrun_override = minrun > MAX_MINRUN ? MAX_MINRUN : minrun; }

void vmps_test_set_tiles(uint32_t fuse_z, uint32_t merge_tile, uint32_t block_elems) {
  if (fuse_z) fuse_z = std::min<uint32_t>(std::max<uint32_t>(fuse_z, 64), MAX_FUSE_Z);
  if (merge_tile) merge_tile = std::min<uint32_t>(std::max<uint32_t>(merge_tile, 16), DEFAULT_TOUT);
  g_fuse_z = fuse_z;
  g_tout = merge_tile;
  g_blk = block_elems;
}

}  // extern "C"

// ===========================================================================
// Multi-GPU building blocks: rank counting and merging of sorted runs.
// ===========================================================================
namespace vmps {

template <int KT>
__global__ void k_count_rank(const typename KeyTraits<KT>::K* __restrict__ keys, uint32_t n,
                             const uint64_t* __restrict__ probes, uint32_t np,
                             unsigned long long* __restrict__ lt, unsigned long long* __restrict__ le) {
  using T = KeyTraits<KT>;
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const uint64_t v = probes[p];
  uint32_t a = 0, b = n;  // first x with img >= v
  while (a < b) { uint32_t m = (a + b) >> 1; if ((uint64_t)T::ord(keys[m]) < v) a = m + 1; else b = m; }
  lt[p] = a;
  b = n;  // first x with img > v (from a on)
  while (a < b) { uint32_t m = (a + b) >> 1; if ((uint64_t)T::ord(keys[m]) <= v) a = m + 1; else b = m; }
  le[p] = a;
}

// Host description of a balanced merge tree over nruns sorted runs.
struct MRLayout {
  uint32_t m;       // runs
  uint32_t H;       // tree height
  size_t off_rs, off_segl, off_segr, off_dep, off_lnodes, off_ltiles, off_lstart, off_ltile,
      off_longs, off_longoff, off_scalars, off_desc, off_k1, off_v1, total;
  uint32_t part_cap;
};

static MRLayout mr_layout(uint64_t n, int kt, int hv, uint32_t m) {
  MRLayout L;
  memset(&L, 0, sizeof(L));
  L.m = m;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align_up(bytes); return o; };
  const size_t R = (size_t)m + 2;
  L.off_k1 = take(n * key_bytes(kt));
  L.off_v1 = hv ? take(n * 4) : 0;
  L.off_rs = take(R * 4);
  L.off_segl = take(R * 4);
  L.off_segr = take(R * 4);
  L.off_dep = take(R * 4);
  L.off_lnodes = take(R * 4);
  L.off_ltiles = take(R * 4);
  L.off_lstart = take((LEVEL_SLOTS + 1) * 4);
  L.off_ltile = take((LEVEL_SLOTS + 1) * 4);
  L.off_longs = take(R * 4 * 4);
  L.off_longoff = take(R * 4);
  L.off_scalars = take(SC_COUNT * 4 + 64);
  L.part_cap = (uint32_t)(n / DEFAULT_TOUT + 2 * (size_t)m + 8);
  L.off_desc = take((size_t)L.part_cap * sizeof(TileDesc));
  L.total = off;
  return L;
}

template <int KT, bool HV>
static vmps_status_t merge_runs_impl(void* keys, uint32_t* vals, uint64_t n, const uint64_t* h_rs,
                                     uint32_t m, char* base, cudaStream_t s) {
  using K = typename KeyTraits<KT>::K;
  MRLayout L = mr_layout(n, KT, HV ? 1 : 0, m);
  const size_t R = (size_t)m + 2;
  // ---- build the tree on the host (balanced split at the middle run) ----
  std::vector<uint32_t> rs(R, 0), segl(R, 0), segr(R, 0), dep(R, 0), height(R, 0);
  for (uint32_t t = 0; t < m; ++t) rs[t] = (uint32_t)h_rs[t];
  rs[m] = (uint32_t)n;
  std::vector<uint32_t> leaf_depth(m, 0);
  struct Frame { uint32_t lo, hi, depth; };
  // recursive build via explicit post-order to compute heights
  std::vector<uint32_t> order;  // internal nodes in post-order
  std::function<uint32_t(uint32_t, uint32_t, uint32_t)> build = [&](uint32_t lo, uint32_t hi, uint32_t d) -> uint32_t {
    if (hi - lo == 1) { leaf_depth[lo] = d; return 0; }
    uint32_t mid = (lo + hi) / 2;
    uint32_t h1 = build(lo, mid, d + 1), h2 = build(mid, hi, d + 1);
    segl[mid] = lo; segr[mid] = hi; dep[mid] = d & 1u;
    height[mid] = 1 + std::max(h1, h2);
    order.push_back(mid);
    return height[mid];
  };
  uint32_t H = build(0, m, 0);
  L.H = H;
  if (H + 2 > (uint32_t)LEVEL_SLOTS) { g_err = "merge_runs: too many runs"; return VMPS_ERR_INVALID_ARG; }
  std::vector<uint32_t> lnodes, ltiles, lstart(LEVEL_SLOTS + 1, 0), ltile(LEVEL_SLOTS + 1, 0);
  for (uint32_t h = 0; h <= (uint32_t)LEVEL_SLOTS - 1; ++h) {
    lstart[h] = (uint32_t)lnodes.size();
    for (uint32_t t : order) if (height[t] == h) lnodes.push_back(t);
  }
  lstart[LEVEL_SLOTS] = (uint32_t)lnodes.size();
  uint32_t acc = 0;
  for (uint32_t x = 0; x < lnodes.size(); ++x) {
    ltiles.push_back(acc);
    uint32_t t = lnodes[x];
    uint32_t i = rs[segl[t]], k = rs[segr[t]];
    acc += (k + DEFAULT_TOUT - 1) / DEFAULT_TOUT - i / DEFAULT_TOUT;
  }
  ltiles.push_back(acc);
  for (uint32_t h = 0; h <= (uint32_t)LEVEL_SLOTS; ++h) ltile[h] = ltiles[lstart[h]];
  // odd-depth leaves start in buffer 1 (copied there by the long-leaf kernel)
  std::vector<uint32_t> longs, longoff;
  uint32_t nlong = 0, chunks = 0;
  for (uint32_t t = 0; t < m; ++t) {
    if (leaf_depth[t] & 1u) {
      uint32_t a = rs[t], e = rs[t + 1];
      longs.push_back(a); longs.push_back(e); longs.push_back(1u); longs.push_back(0u);
      longoff.push_back(chunks);
      chunks += (e - a + LONG_CHUNK - 1) / LONG_CHUNK;
      ++nlong;
    }
  }
  longoff.push_back(chunks);
  std::vector<uint32_t> scal(SC_COUNT, 0);
  scal[SC_LONG] = nlong;
  // ---- upload ----
  auto up = [&](size_t off, const void* src, size_t bytes) -> cudaError_t {
    if (!bytes) return cudaSuccess;
    return cudaMemcpyAsync(base + off, src, bytes, cudaMemcpyHostToDevice, s);
  };
  VMPS_CK(up(L.off_rs, rs.data(), R * 4));
  VMPS_CK(up(L.off_segl, segl.data(), R * 4));
  VMPS_CK(up(L.off_segr, segr.data(), R * 4));
  VMPS_CK(up(L.off_dep, dep.data(), R * 4));
  VMPS_CK(up(L.off_lnodes, lnodes.data(), lnodes.size() * 4));
  VMPS_CK(up(L.off_ltiles, ltiles.data(), ltiles.size() * 4));
  VMPS_CK(up(L.off_lstart, lstart.data(), lstart.size() * 4));
  VMPS_CK(up(L.off_ltile, ltile.data(), ltile.size() * 4));
  VMPS_CK(up(L.off_longs, longs.data(), longs.size() * 4));
  VMPS_CK(up(L.off_longoff, longoff.data(), longoff.size() * 4));
  VMPS_CK(up(L.off_scalars, scal.data(), SC_COUNT * 4));
  VMPS_CK(cudaStreamSynchronize(s));  // host vectors die at return
  K* k0 = (K*)keys;
  K* k1 = (K*)(base + L.off_k1);
  uint32_t* v0 = vals;
  uint32_t* v1 = HV ? (uint32_t*)(base + L.off_v1) : nullptr;
  uint32_t* d_scal = (uint32_t*)(base + L.off_scalars);
  LAUNCH((k_long_leaves<KT, HV>), nsm() * VMPS_LONG_MINB, 256, 0, s, k0, v0, k1, v1, (const uint32_t*)(base + L.off_longs),
         (const uint32_t*)(base + L.off_longoff), d_scal, LONG_CHUNK);
  using SM = MergeSmem<KT, HV>;
  VMPS_CK(cudaFuncSetAttribute(k_merge_level<KT, HV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::BYTES));
  int occ = 0;
  VMPS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_merge_level<KT, HV>, MERGE_BLOCK, SM::BYTES));
  const unsigned gm = (unsigned)(nsm() * (occ > 0 ? occ : 1));
  TileDesc* desc = (TileDesc*)(base + L.off_desc);
  for (uint32_t h = 1; h <= H; ++h) {
    LAUNCH(k_tile_desc<KT>, (L.part_cap + 255) / 256, 256, 0, s, k0, k1, (const uint32_t*)(base + L.off_rs),
           (const uint32_t*)(base + L.off_segl), (const uint32_t*)(base + L.off_segr),
           (const uint32_t*)(base + L.off_dep), (const uint32_t*)(base + L.off_lnodes),
           (const uint32_t*)(base + L.off_ltiles), (const uint32_t*)(base + L.off_lstart),
           (const uint32_t*)(base + L.off_ltile), (int)h, (uint32_t)DEFAULT_TOUT, desc, L.part_cap, d_scal);
    LAUNCH((k_merge_level<KT, HV>), gm, MERGE_BLOCK, SM::BYTES, s, k0, v0, k1, v1, desc,
           (const uint32_t*)(base + L.off_ltile), (int)h, (uint32_t)DEFAULT_TOUT, L.part_cap);
  }
  return launch_check();
}

}  // namespace vmps

extern "C" {

vmps_status_t vmps_count_rank(const void* keys, uint64_t n, vmps_key_t kt, const uint64_t* probes,
                              uint32_t nprobe, uint64_t* out_lt, uint64_t* out_le, void* stream) {
  vmps_status_t rc = check_common(keys, nullptr, n, kt);
  if (rc != VMPS_OK) return rc;
  if (nprobe == 0) return VMPS_OK;
  if (!probes || !out_lt || !out_le) { g_err = "NULL probe/output"; return VMPS_ERR_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned g = (nprobe + 127) / 128;
  switch (kt) {
    case VMPS_KEY_U32:
      k_count_rank<VMPS_KEY_U32><<<g, 128, 0, s>>>((const uint32_t*)keys, (uint32_t)n, probes, nprobe,
                                                   (unsigned long long*)out_lt, (unsigned long long*)out_le);
      break;
    case VMPS_KEY_U64:
      k_count_rank<VMPS_KEY_U64><<<g, 128, 0, s>>>((const uint64_t*)keys, (uint32_t)n, probes, nprobe,
                                                   (unsigned long long*)out_lt, (unsigned long long*)out_le);
      break;
    default:
      k_count_rank<VMPS_KEY_F32><<<g, 128, 0, s>>>((const uint32_t*)keys, (uint32_t)n, probes, nprobe,
                                                   (unsigned long long*)out_lt, (unsigned long long*)out_le);
  }
  ++g_nl;
  return launch_check();
}

// ---- pull-merge of pieces at arbitrary addresses ----
}  // extern "C"
namespace vmps {
template <int KT, bool HV>
static vmps_status_t pull_pass(const void* const* kp, const uint32_t* const* vp, const uint64_t* cnt, uint32_t g,
                               void* ok, uint32_t* ov, uint32_t base, TileDesc4* tiles, cudaStream_t s) {
  using K = typename KeyTraits<KT>::K;
  using SM4 = Merge4Smem<KT, HV>;
  PullSrc<KT> S;
  uint64_t N = 0;
  for (int i = 0; i < 4; ++i) {
    const bool on = (uint32_t)i < g && cnt[i] > 0;
    S.kp[i] = on ? (const K*)kp[i] : nullptr;
    S.vp[i] = (on && HV) ? vp[i] : nullptr;
    S.n[i] = on ? (uint32_t)cnt[i] : 0u;
    N += S.n[i];
  }
  S.N = (uint32_t)N;
  S.base = base;
  if (N == 0) return VMPS_OK;
  static int occ_t[MAX_DEV][3][2] = {};
  auto& occ = occ_t[dev_slot()];
  if (!occ[KT][HV]) {
    VMPS_CK(cudaFuncSetAttribute(k_pull_merge<KT, HV, M4_KQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SM4::BYTES));
    int o = 0;
    VMPS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_pull_merge<KT, HV, M4_KQ>, M4_THREADS,
                                                          SM4::BYTES));
    occ[KT][HV] = o > 0 ? o : 1;
  }
  const uint32_t ntiles = (uint32_t)((base + N + 4095) / 4096 - base / 4096);
  const uint32_t nchunks = (ntiles + DESC4_CHUNK - 1) / DESC4_CHUNK;
  LAUNCH(k_pull_desc<KT>, (nchunks + 255) / 256, 256, 0, s, S, ntiles, tiles);
  LAUNCH((k_pull_merge<KT, HV, M4_KQ>), (unsigned)std::min<uint32_t>(ntiles, nsm() * occ[KT][HV]),
         M4_THREADS, SM4::BYTES, s, S, (K*)ok, ov, tiles, ntiles);
  return launch_check();
}

template <int KT, bool HV>
static vmps_status_t pull_dispatch(const void* const* kp, const uint32_t* const* vp, const uint64_t* cnt,
                                   uint32_t g, void* ok, uint32_t* ov, uint32_t base, TileDesc4* tiles,
                                   cudaStream_t s) {
  return pull_pass<KT, HV>(kp, vp, cnt, g, ok, ov, base, tiles, s);
}
}  // namespace vmps
extern "C" {

vmps_status_t vmps_merge_pieces_workspace_bytes(uint64_t n_total, vmps_key_t kt, int has_vals, uint32_t g,
                                                size_t* h_bytes) {
  if (!h_bytes || g < 1 || g > 8 || n_total > VMPS_MAX_N) return VMPS_ERR_INVALID_ARG;
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) return VMPS_ERR_INVALID_ARG;
  size_t b = align_up(((size_t)(n_total + 4095) / 4096 + 2) * sizeof(TileDesc4));
  if (g > 4 && n_total > 1) {
    size_t m = 0;
    if (vmps_merge_runs_workspace_bytes(n_total, kt, has_vals, 2, &m) != VMPS_OK) return VMPS_ERR_INVALID_ARG;
    b += align_up(m);
  }
  *h_bytes = b + 256;
  return VMPS_OK;
}

vmps_status_t vmps_merge_pieces(const void* const* h_keys, const uint32_t* const* h_vals, const uint64_t* h_counts,
                                uint32_t g, void* out_keys, uint32_t* out_vals, vmps_key_t kt, void* ws,
                                size_t ws_bytes, void* stream) {
  if (!h_keys || !h_counts || g < 1 || g > 8) { g_err = "pieces: need 1..8 pieces"; return VMPS_ERR_INVALID_ARG; }
  uint64_t N = 0;
  for (uint32_t i = 0; i < g; ++i) {
    if (h_counts[i] && (!h_keys[i] || (out_vals && (!h_vals || !h_vals[i])))) {
      g_err = "pieces: NULL piece pointer";
      return VMPS_ERR_INVALID_ARG;
    }
    N += h_counts[i];
  }
  vmps_status_t rc = check_common(out_keys, out_vals, N, kt);
  if (rc != VMPS_OK) return rc;
  size_t need = 0;
  if (vmps_merge_pieces_workspace_bytes(N, kt, out_vals ? 1 : 0, g, &need) != VMPS_OK) return VMPS_ERR_INVALID_ARG;
  if (!ws || ws_bytes < need) { g_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  if (N == 0) return VMPS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  TileDesc4* tiles = (TileDesc4*)base;
  const size_t tb = align_up(((size_t)(N + 4095) / 4096 + 2) * sizeof(TileDesc4));  // >= tiles of either pass
  const uint32_t* vnull[8] = {nullptr};
  const uint32_t* const* vp = out_vals ? h_vals : vnull;
  const size_t kb = key_bytes(kt);
  uint64_t N1 = 0;
  for (uint32_t i = 0; i < std::min<uint32_t>(g, 4); ++i) N1 += h_counts[i];
  for (uint32_t part = 0; part < (g > 4 ? 2u : 1u); ++part) {
    const uint32_t i0 = 4 * part, gg = std::min<uint32_t>(g - i0, 4);
    // both passes write through the (aligned) output base; the second one's
    // tiles start at position N1
    char* okp = (char*)out_keys;
    uint32_t* ovp = out_vals;
    const uint32_t obase = part ? (uint32_t)N1 : 0u;
    (void)kb;
    if (out_vals) {
      switch (kt) {
        case VMPS_KEY_U32: rc = pull_dispatch<VMPS_KEY_U32, true>(h_keys + i0, vp + i0, h_counts + i0, gg, okp, ovp, obase, tiles, s); break;
        case VMPS_KEY_U64: rc = pull_dispatch<VMPS_KEY_U64, true>(h_keys + i0, vp + i0, h_counts + i0, gg, okp, ovp, obase, tiles, s); break;
        default: rc = pull_dispatch<VMPS_KEY_F32, true>(h_keys + i0, vp + i0, h_counts + i0, gg, okp, ovp, obase, tiles, s); break;
      }
    } else {
      switch (kt) {
        case VMPS_KEY_U32: rc = pull_dispatch<VMPS_KEY_U32, false>(h_keys + i0, vp + i0, h_counts + i0, gg, okp, nullptr, obase, tiles, s); break;
        case VMPS_KEY_U64: rc = pull_dispatch<VMPS_KEY_U64, false>(h_keys + i0, vp + i0, h_counts + i0, gg, okp, nullptr, obase, tiles, s); break;
        default: rc = pull_dispatch<VMPS_KEY_F32, false>(h_keys + i0, vp + i0, h_counts + i0, gg, okp, nullptr, obase, tiles, s); break;
      }
    }
    if (rc != VMPS_OK) return rc;
  }
  if (g > 4 && N1 > 0 && N1 < N) {
    const uint64_t st2[2] = {0, N1};
    return vmps_merge_runs(out_keys, out_vals, N, kt, st2, 2, base + tb, ws_bytes - (size_t)(base - (char*)ws) - tb,
                           stream);
  }
  return VMPS_OK;
}

vmps_status_t vmps_merge_runs_workspace_bytes(uint64_t n, vmps_key_t kt, int has_vals, uint32_t nruns,
                                              size_t* h_bytes) {
  if (!h_bytes || nruns == 0) return VMPS_ERR_INVALID_ARG;
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) return VMPS_ERR_INVALID_ARG;
  if (n > VMPS_MAX_N) return VMPS_ERR_INVALID_ARG;
  *h_bytes = mr_layout(n, kt, has_vals ? 1 : 0, nruns).total + 256;
  return VMPS_OK;
}

vmps_status_t vmps_merge_runs(void* keys, uint32_t* vals, uint64_t n, vmps_key_t kt, const uint64_t* h_run_start,
                              uint32_t nruns, void* ws, size_t ws_bytes, void* stream) {
  vmps_status_t rc = check_common(keys, vals, n, kt);
  if (rc != VMPS_OK) return rc;
  if (!h_run_start || nruns == 0) { g_err = "no runs"; return VMPS_ERR_INVALID_ARG; }
  if (h_run_start[0] != 0) { g_err = "run_start[0] must be 0"; return VMPS_ERR_INVALID_ARG; }
  for (uint32_t t = 1; t < nruns; ++t)
    if (h_run_start[t] <= h_run_start[t - 1] || h_run_start[t] >= n) {
      g_err = "run starts must be strictly increasing and < n";
      return VMPS_ERR_INVALID_ARG;
    }
  if (nruns == 1 || n <= 1) return VMPS_OK;
  const int hv = vals ? 1 : 0;
  MRLayout L = mr_layout(n, kt, hv, nruns);
  char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if (!ws || (size_t)(base - (char*)ws) + L.total > ws_bytes) { g_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  cudaStream_t s = (cudaStream_t)stream;
  switch (kt) {
    case VMPS_KEY_U32:
      return hv ? merge_runs_impl<VMPS_KEY_U32, true>(keys, vals, n, h_run_start, nruns, base, s)
                : merge_runs_impl<VMPS_KEY_U32, false>(keys, vals, n, h_run_start, nruns, base, s);
    case VMPS_KEY_U64:
      return hv ? merge_runs_impl<VMPS_KEY_U64, true>(keys, vals, n, h_run_start, nruns, base, s)
                : merge_runs_impl<VMPS_KEY_U64, false>(keys, vals, n, h_run_start, nruns, base, s);
    default:
      return hv ? merge_runs_impl<VMPS_KEY_F32, true>(keys, vals, n, h_run_start, nruns, base, s)
                : merge_runs_impl<VMPS_KEY_F32, false>(keys, vals, n, h_run_start, nruns, base, s);
  }
}

}  // extern "C"
