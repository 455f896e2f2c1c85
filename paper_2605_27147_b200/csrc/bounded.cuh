// bounded.cuh -- scratch-bounded mode (BASELINE.json north_star (4); SURVEY
// 8(a) A9): element scratch capped at S = c sqrt(n log2 n) elements.
//
// The array is cut into blocks of P elements.  Physical blocks are the
// caller's blocks 0..NB-1 plus F = floor(S / P) scratch blocks NB..NB+F-1; the
// block table T_in maps virtual block v (positions [vP, vP+P)) to the
// physical block holding it (the paper's page lists, as one array,
// App. A).  Leaves are sorted in place.  Each tree level is then a
// left-to-right stream of output blocks: a round takes free physical blocks
// for the next dirty output blocks (T_out), runs their tiles -- merge tiles of
// the level's nodes and copy tiles for the other elements of those blocks --
// and every tile subtracts the elements it consumed from per-block counters;
// a block whose counter reaches zero goes back to the free pool (a consumed
// page is released and reused as output, Fig. 2).  At the end
// the blocks are permuted into physical order with evictions (Copy).
#pragma once
#include "engine.cuh"
#include "plan.cuh"
#include "ptx.cuh"
#include <cooperative_groups.h>

namespace vmps {
namespace cg = cooperative_groups;

constexpr uint32_t BD_NONE = 0xFFFFFFFFu;

struct BdState {          // device-side state (one per sort)
  uint32_t head, tail;    // free-block ring (pool[x % cap]) during the levels
  uint32_t ticket;        // next dirty output block of the level
  uint32_t err;           // 1 = no free block (budget too small)
  uint32_t pool_count;    // Copy: free blocks in pool[0, pool_count)
  uint32_t rounds;        // level passes that moved data (statistics)
  uint32_t copies;        // final Copy: block copies
  uint32_t copy_q;        // final Copy: virtual blocks [0, copy_q) are home
};

template <int KT>
struct BdMem {
  using K = typename KeyTraits<KT>::K;
  K* k0; uint32_t* v0;    // caller's array
  K* ks; uint32_t* vs;    // scratch blocks
  uint32_t NB, P, n, has_partial;
  uint32_t lg;            // log2 P (P is a power of two)
  __device__ __forceinline__ K* kb(uint32_t b) const {
    return b < NB ? k0 + ((size_t)b << lg) : ks + ((size_t)(b - NB) << lg);
  }
  __device__ __forceinline__ uint32_t* vb(uint32_t b) const {
    return b < NB ? v0 + ((size_t)b << lg) : vs + ((size_t)(b - NB) << lg);
  }
  __device__ __forceinline__ uint32_t vlen(uint32_t v) const {  // elements of virtual block v
    return v + 1 < NB ? P : n - (v << lg);
  }
};

// --- per-level setup ------------------------------------------------------
// --- the call's level schedule, built once --------------------------------
// The non-fused nodes (segment > fuse_z) bucketed by power, in position order
// inside each bucket (a stable counting sort: per-tile histograms, one scan in
// bucket-major order, a stable scatter), so that level p is the slice
// [hscan[p T], hscan[(p + 1) T]) of lnodes (T tiles of 1024 boundaries).
constexpr uint32_t BD_LVL_TILE = 1024;
constexpr uint32_t BD_LVL_BINS = 64;

__device__ __forceinline__ uint32_t bd_node_bin(const uint32_t* rs, const uint32_t* seg_l, const uint32_t* seg_r,
                                                const uint8_t* power, uint32_t r, uint32_t fuse_z, uint32_t t) {
  if (t < 1 || t >= r) return BD_LVL_BINS;
  return seg_size(rs, seg_l, seg_r, t) > fuse_z ? (uint32_t)power[t] : BD_LVL_BINS;
}

__global__ void __launch_bounds__(BD_LVL_TILE) k_lvl_hist(const uint32_t* __restrict__ rs, const uint32_t* scalars,
                                                          const uint8_t* __restrict__ power,
                                                          const uint32_t* __restrict__ seg_l,
                                                          const uint32_t* __restrict__ seg_r, uint32_t fuse_z,
                                                          uint32_t ntiles, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[BD_LVL_BINS];
  const uint32_t r = scalars[SC_RUNS];
  if (threadIdx.x < BD_LVL_BINS) h[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t t = blockIdx.x * BD_LVL_TILE + threadIdx.x;
  const uint32_t bin = bd_node_bin(rs, seg_l, seg_r, power, r, fuse_z, t);
  if (bin < BD_LVL_BINS) atomicAdd(&h[bin], 1u);
  __syncthreads();
  if (threadIdx.x < BD_LVL_BINS) hist[threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
  if (blockIdx.x == 0 && threadIdx.x == 0) hist[BD_LVL_BINS * ntiles] = 0;  // the scan's total slot
}

__global__ void __launch_bounds__(BD_LVL_TILE) k_lvl_scatter(const uint32_t* __restrict__ rs, const uint32_t* scalars,
                                                             const uint8_t* __restrict__ power,
                                                             const uint32_t* __restrict__ seg_l,
                                                             const uint32_t* __restrict__ seg_r, uint32_t fuse_z,
                                                             uint32_t ntiles, const uint32_t* __restrict__ hscan,
                                                             uint32_t* __restrict__ lnodes) {
  __shared__ uint32_t wc[BD_LVL_TILE / 32][BD_LVL_BINS];  // per-warp bucket counts
  const uint32_t r = scalars[SC_RUNS];
  const uint32_t lane = threadIdx.x & 31u, wp = threadIdx.x >> 5;
  for (uint32_t x = threadIdx.x; x < (BD_LVL_TILE / 32) * BD_LVL_BINS; x += BD_LVL_TILE) (&wc[0][0])[x] = 0;
  __syncthreads();
  const uint32_t t = blockIdx.x * BD_LVL_TILE + threadIdx.x;
  const uint32_t bin = bd_node_bin(rs, seg_l, seg_r, power, r, fuse_z, t);
  const uint32_t peers = __match_any_sync(0xFFFFFFFFu, bin);
  const uint32_t rank = (uint32_t)__popc(peers & ((1u << lane) - 1u));
  if (bin < BD_LVL_BINS && rank == 0) wc[wp][bin] = (uint32_t)__popc(peers);
  __syncthreads();
  if (bin < BD_LVL_BINS) {
    uint32_t pos = hscan[bin * ntiles + blockIdx.x] + rank;
    for (uint32_t w = 0; w < wp; ++w) pos += wc[w][bin];
    lnodes[pos] = t;
  }
}

// Tile counts of every bucketed node (neighbours only within its level) and,
// per level pass, the level's slice: info = {ls, m, first tile, tiles}.
__device__ __forceinline__ void bd_level_of(const uint32_t* hscan, uint32_t ntiles, uint32_t x, uint32_t* ls,
                                            uint32_t* le) {
  uint32_t lo = 0, hi = BD_LVL_BINS;  // last bin p with hscan[p T] <= x
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (hscan[mid * ntiles] <= x) lo = mid;
    else hi = mid;
  }
  while (lo + 1 < BD_LVL_BINS && hscan[(lo + 1) * ntiles] <= x) ++lo;  // skip empty bins
  *ls = hscan[lo * ntiles];
  *le = hscan[(lo + 1) * ntiles];
}

__device__ __forceinline__ void bd_node_geom(const uint32_t* rs, const uint32_t* seg_l, const uint32_t* seg_r,
                                             const uint32_t* lnodes, uint32_t m, uint32_t x, uint32_t P,
                                             uint32_t n, uint32_t* i, uint32_t* j, uint32_t* k,
                                             uint32_t* lgap_lo, uint32_t* rgap_hi) {
  const uint32_t t = lnodes[x];
  *i = rs[seg_l[t]];
  *j = rs[t];
  *k = rs[seg_r[t]];
  const uint32_t bs = (*i / P) * P;                                  // first block start
  const uint32_t kprev = x > 0 ? rs[seg_r[lnodes[x - 1]]] : 0u;
  *lgap_lo = (bs < *i && kprev <= bs) ? bs : *i;                     // [lgap_lo, i) copy tile
  const uint32_t be = min(n, ((*k + P - 1) / P) * P);                // last block end
  const uint32_t inext = x + 1 < m ? rs[seg_l[lnodes[x + 1]]] : n;
  *rgap_hi = max(*k, min(be, inext));                                // [k, rgap_hi) copy tile
}

__global__ void k_bd_tile_counts(const uint32_t* __restrict__ rs, const uint32_t* __restrict__ seg_l,
                                 const uint32_t* __restrict__ seg_r, const uint32_t* __restrict__ lnodes,
                                 const uint32_t* __restrict__ hscan, uint32_t ntiles, uint32_t P, uint32_t n,
                                 uint32_t cap, uint32_t* __restrict__ cnt) {
  const uint32_t X = hscan[BD_LVL_BINS * ntiles];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= cap; x += gridDim.x * blockDim.x) {
    uint32_t c = 0;
    if (x < X) {
      uint32_t ls, le, i, j, k, gl, gh;
      bd_level_of(hscan, ntiles, x, &ls, &le);
      bd_node_geom(rs, seg_l, seg_r, lnodes + ls, le - ls, x - ls, P, n, &i, &j, &k, &gl, &gh);
      c = (k + P - 1) / P - i / P + (gl < i ? 1u : 0u) + (gh > k ? 1u : 0u);
    }
    cnt[x] = c;
  }
}

// Translated key load: virtual position q through the block table.
template <int KT>
__device__ __forceinline__ typename KeyTraits<KT>::K bd_key(const BdMem<KT>& M, const uint32_t* Tin,
                                                            uint32_t q) {
  return M.kb(Tin[q >> M.lg])[q & (M.P - 1)];
}

#ifndef VMPS_BD_RF
#define VMPS_BD_RF 1
#endif
template <int KT>
__device__ uint32_t bd_corank(const BdMem<KT>& M, const uint32_t* Tin, uint32_t ai, uint32_t nA, uint32_t bi,
                              uint32_t nB, uint32_t d) {
  using T = KeyTraits<KT>;
  uint32_t lo = d > nB ? d - nB : 0u, hi = min(d, nA);
  if constexpr (VMPS_BD_RF) {  // regula falsi steps (RFalsi, engine4.cuh): exact, fewer dependent probes
    RFalsi rf;
    rf.init();
    while (lo < hi) {
      bool interp;
      const uint32_t mid = rf.probe(lo, hi, &interp), w0 = hi - lo;
      const auto a = bd_key<KT>(M, Tin, ai + mid), b = bd_key<KT>(M, Tin, bi + d - mid - 1);
      const bool p = T::ord(a) <= T::ord(b);
      if (p) lo = mid + 1;
      else hi = mid;
      rf.update(p, interp_gap<KT>(a, b), w0, hi - lo, interp);
    }
    return lo;
  } else {
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (T::ord(bd_key<KT>(M, Tin, ai + mid)) <= T::ord(bd_key<KT>(M, Tin, bi + d - mid - 1))) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  }
}

// A tile of a bounded level pass: output positions [lo, hi) of the node
// [i, k) whose runs are [i, j) and [j, k); a0 / a1 = elements of [i, j)
// among the node's first lo - i / hi - i outputs.  A gap tile (copy of the
// elements between nodes) is a node with an empty right run.  (k is not
// needed once the tile is cut: 24 bytes per tile.)
struct BdTile {
  uint32_t i, j, lo, hi, a0, a1;
};

// Tile descriptors of the level in output order (one thread per tile), and
// the dirty output blocks.  A merge tile is an identity when every element it
// outputs already sits at its output position: the whole node is a
// concatenation (A's last <= B's first), or the tile takes only A elements
// with no B element before it, or only B elements after all of A (the page
// hand-over of P:514-515 in its in-place form).  A block is dirty iff a
// non-identity merge tile writes into it; a clean block keeps its physical
// home and its tiles are skipped: zero bytes moved.  (An element that leaves
// a block makes that block's own output differ there, so dirty blocks only
// ever consume inputs from dirty blocks.)  The level's slice of the schedule
// (info: first node, nodes, first tile, tiles) is read here and published
// for the later kernels of the pass.
template <int KT>
__global__ void __launch_bounds__(256) k_bd_tile_desc(BdMem<KT> M, const uint32_t* __restrict__ Tin,
                                                      const uint32_t* __restrict__ rs,
                                                      const uint32_t* __restrict__ seg_l,
                                                      const uint32_t* __restrict__ seg_r,
                                                      const uint32_t* __restrict__ lnodes_all,
                                                      const uint32_t* __restrict__ hscan, uint32_t nlt, int p,
                                                      const uint32_t* __restrict__ toff_all, uint32_t cap,
                                                      BdState* st, BdTile* __restrict__ desc,
                                                      uint32_t* __restrict__ info, uint32_t vb0,
                                                      uint32_t* __restrict__ dirty) {
  using T = KeyTraits<KT>;
  const uint32_t ls = hscan[(uint32_t)p * nlt], le = hscan[(uint32_t)(p + 1) * nlt];
  const uint32_t m = le - ls, T0 = toff_all[ls], total = toff_all[le] - T0;
  if (blockIdx.x == 0 && threadIdx.x == 0) { info[0] = ls; info[1] = m; info[2] = T0; info[3] = total; }
  const uint32_t* lnodes = lnodes_all + ls;
  const uint32_t* toff = toff_all + ls;
  if (total > cap) {  // capacity is sized from the plan; never expected
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(&st->err, 2u);
    return;
  }
  const uint32_t P = M.P, n = M.n;
  for (uint32_t tau = blockIdx.x * blockDim.x + threadIdx.x; tau < total; tau += gridDim.x * blockDim.x) {
    uint32_t a = 0, b = m;  // last node x with toff[x] - T0 <= tau
    while (b - a > 1) { uint32_t mm = (a + b) >> 1; if (toff[mm] - T0 <= tau) a = mm; else b = mm; }
    uint32_t i, j, k, gl, gh;
    bd_node_geom(rs, seg_l, seg_r, lnodes, m, a, P, n, &i, &j, &k, &gl, &gh);
    uint32_t loc = tau - (toff[a] - T0);
    BdTile D;
    if (gl < i && loc == 0) {  // left gap: copy [gl, i) (an identity: moves only with a dirty block)
      D.i = gl; D.j = i; D.lo = gl; D.hi = i; D.a0 = 0; D.a1 = i - gl;
      desc[tau] = D;
      continue;
    }
    if (gl < i) --loc;
    const uint32_t nt = (k + P - 1) / P - i / P;
    if (loc >= nt) {  // right gap: copy [k, gh)
      D.i = k; D.j = gh; D.lo = k; D.hi = gh; D.a0 = 0; D.a1 = gh - k;
      desc[tau] = D;
      continue;
    }
    const uint32_t g = i / P + loc;
    const uint32_t lo = max(i, g * P), hi = min(k, (g + 1) * P);
    const uint32_t nA = j - i, nB = k - j;
    const uint32_t a0 = lo == i ? 0u : bd_corank<KT>(M, Tin, i, nA, j, nB, lo - i);
    const uint32_t a1 = hi == k ? nA : bd_corank<KT>(M, Tin, i, nA, j, nB, hi - i);
    D.i = i; D.j = j; D.lo = lo; D.hi = hi; D.a0 = a0; D.a1 = a1;
    desc[tau] = D;
    const uint32_t nAt = a1 - a0, nBt = (hi - lo) - nAt, b0 = (lo - i) - a0;
    bool ident = (nBt == 0 && b0 == 0) || (nAt == 0 && a0 == nA);
    if (!ident && nA > 0 && nB > 0) ident = T::ord(bd_key<KT>(M, Tin, j - 1)) <= T::ord(bd_key<KT>(M, Tin, j));
    if (!ident) dirty[lo / P - vb0] = 1u;
  }
}

// Small passes (a block range up to BD_SMALL_MAX): the scan of the dirty
// flags, the dirty list, first tiles, consumption counters and count, by one
// CTA of 1024 threads in place of the scan launches + k_bd_dirty_list.
constexpr uint32_t BD_SMALL_THREADS = 1024;
constexpr uint32_t BD_SMALL_MAX = 32768;
template <int KT>
__global__ void __launch_bounds__(BD_SMALL_THREADS) k_bd_dirty_small(
    BdMem<KT> M, const BdTile* __restrict__ desc, const uint32_t* __restrict__ info,
    const uint32_t* __restrict__ dirty, uint32_t* __restrict__ didx, uint32_t vb0, uint32_t nbr,
    uint32_t* __restrict__ dlist, uint32_t* __restrict__ first_tile, uint32_t* __restrict__ remain,
    uint32_t* __restrict__ D_out) {
  __shared__ uint32_t wsum[BD_SMALL_THREADS / 32];
  __shared__ uint32_t s_carry[2];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid == 0) s_carry[0] = 0;
  __syncthreads();
  uint32_t it = 0;
  for (uint32_t base = 0; base < nbr; base += BD_SMALL_THREADS, ++it) {
    const uint32_t x = base + tid;
    const uint32_t f = x < nbr ? dirty[x] : 0u;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f != 0u);
    if (lane == 0) wsum[warp] = (uint32_t)__popc(bal);
    __syncthreads();
    const uint32_t carry = s_carry[it & 1u];
    if (warp == 0) {
      const uint32_t w = wsum[lane];
      uint32_t incl = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)lane >= o) incl += y;
      }
      wsum[lane] = incl - w;
      if (lane == 31) s_carry[(it + 1u) & 1u] = carry + incl;
    }
    __syncthreads();
    if (f) {
      const uint32_t idx = carry + wsum[warp] + (uint32_t)__popc(bal & ((1u << lane) - 1u));
      didx[x] = idx;
      dlist[idx] = vb0 + x;
      remain[vb0 + x] = M.vlen(vb0 + x);
    }
    __syncthreads();
  }
  const uint32_t total = info[3], P = M.P, D = s_carry[it & 1u];
  for (uint32_t tau = tid; tau < total; tau += BD_SMALL_THREADS) {
    const uint32_t x = desc[tau].lo / P - vb0;
    if (dirty[x] && (tau == 0 || desc[tau - 1].lo / P - vb0 != x)) first_tile[didx[x]] = tau;
  }
  if (tid == 0) {
    *D_out = D;
    first_tile[D] = total;
  }
}

// Dirty blocks of the range [vb0, vb0 + nbr) (flags and their scan are
// indexed relative to vb0): their list, first tiles and consumption counters.
template <int KT>
__global__ void k_bd_dirty_list(BdMem<KT> M, const BdTile* __restrict__ desc, const uint32_t* __restrict__ info,
                                const uint32_t* __restrict__ dirty, const uint32_t* __restrict__ didx, uint32_t vb0,
                                uint32_t nbr, uint32_t* __restrict__ dlist, uint32_t* __restrict__ first_tile,
                                uint32_t* __restrict__ remain, uint32_t* __restrict__ D_out) {
  const uint32_t total = info[3];
  const uint32_t P = M.P;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < nbr; x += gridDim.x * blockDim.x) {
    if (dirty[x]) {
      dlist[didx[x]] = vb0 + x;
      remain[vb0 + x] = M.vlen(vb0 + x);
    }
  }
  for (uint32_t tau = blockIdx.x * blockDim.x + threadIdx.x; tau < total; tau += gridDim.x * blockDim.x) {
    const uint32_t x = desc[tau].lo / P - vb0;
    if (dirty[x] && (tau == 0 || desc[tau - 1].lo / P - vb0 != x)) first_tile[didx[x]] = tau;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t D = didx[nbr];
    *D_out = D;
    first_tile[D] = total;
  }
}

// A top merge of the dyadic-cell mode as a two-run plan: runs [0, nx) and
// [nx, len), one node (t = 1) of power 1 covering both.
__global__ void k_bd_top_setup(uint32_t* __restrict__ rs, uint32_t* __restrict__ seg_l, uint32_t* __restrict__ seg_r,
                               uint8_t* __restrict__ power, uint32_t* __restrict__ scalars, uint32_t nx, uint32_t len) {
  if (threadIdx.x == 0) {
    rs[0] = 0; rs[1] = nx; rs[2] = len;
    seg_l[0] = 0; seg_l[1] = 0;
    seg_r[0] = 0; seg_r[1] = 2;
    power[0] = 0; power[1] = 1;
  }
  for (uint32_t i = threadIdx.x; i < SC_COUNT; i += blockDim.x) scalars[i] = i == SC_RUNS ? 2u : 0u;
}

// Run starts of a sub-array made absolute (the shared block table's positions).
__global__ void k_rs_add_base(uint32_t* __restrict__ rs, const uint32_t* scalars, uint32_t base) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= r; t += gridDim.x * blockDim.x) rs[t] += base;
}

// --- level pass: dataflow over the dirty output blocks ---------------------
// One persistent kernel per level.  A CTA takes the next dirty output block
// (ticket), gathers the inputs of all its tiles through T_in into shared
// memory, releases every input block whose elements are now all consumed
// (a consumed page goes back to the free list, Fig. 2), then takes
// a free physical block for its output, merges the tiles in shared memory and
// stores the block.  Free blocks circulate through a ring (pool[x % cap]):
// a release reserves a slot with an atomic on `tail` and publishes the block
// id; an allocation reserves a slot on `head` and waits until it is
// published.  Inputs are released before the allocation, so a level needs no
// more free blocks than the rounds of a block-synchronous schedule would.  A
// CTA that waits ~1 s without a free block reports the budget as too small.
__device__ __forceinline__ uint32_t bd_alloc(BdState* st, uint32_t* pool, uint32_t cap) {
  const uint32_t h = atomicAdd(&st->head, 1u);
  volatile uint32_t* slot = reinterpret_cast<volatile uint32_t*>(pool) + h % cap;
  uint32_t b = *slot;
  if (b == BD_NONE) {
    const long long t0 = clock64();
    while ((b = *slot) == BD_NONE) {
      if (*reinterpret_cast<volatile uint32_t*>(&st->err)) return BD_NONE;
      if (clock64() - t0 > (1ll << 31)) { atomicExch(&st->err, 1u); return BD_NONE; }
      __nanosleep(64);
    }
  }
  *slot = BD_NONE;
  return b;
}

#ifndef VMPS_BD_THREADS
#define VMPS_BD_THREADS 256
#endif
constexpr uint32_t BD_THREADS = VMPS_BD_THREADS;  // threads of a level-pass CTA (MERGE_K outputs each)
constexpr uint32_t BD_MAX_TILES = 32;  // descriptors looked at per output block (at most 3 pieces when P <= Z)

// Per-block header of the level pass: the tiles of one dirty output block,
// the inputs of each tile (part 2x = its A range, 2x+1 = its B range, each of
// <= P elements, so spanning at most two physical blocks) and where each part
// lands in the stage.  A part's keys occupy their own stage region, whose start
// is 16-byte aligned and offset by the part's misalignment in global memory
// (ko = region start + gq mod (16 / sizeof(K))), so that each of its (at most
// two) pieces is ONE bulk copy (cp.async.bulk, TMA engine) of the 16-byte
// aligned superset of the piece; values likewise (vo).
struct BdHdr {
  uint32_t d, v, nt, valid;
  uint32_t nslow;       // pieces gathered element by element (unaligned arrays / the caller's partial last block)
  uint32_t pad[3];
  BdTile t[16];
  uint32_t part[32][2];  // virtual start, length of part x
  uint32_t ko[32], vo[32];  // stage index of part x's first key / value
  uint32_t pcb[32][2];   // physical blocks of part x's two pieces; bit 31: gathered element-wise
};
constexpr uint32_t BD_SLOW = 0x80000000u;

// Slack after each part's region: the superset rounding (< one 16-byte unit
// on either side) plus the branch-free merge's read one past a part's end.
// (V = elements per 16 bytes of the array: 16 / sizeof(K) for keys, 4 for values.)
__host__ __device__ constexpr uint32_t bd_stage_elems(uint32_t P, uint32_t V) { return P + 32u * 3u * V + 64u; }

__device__ __forceinline__ void cp_async_el(void* dst, const void* src, int bytes) {
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Warp 1: take the next dirty output block, read its tiles, resolve the
// physical pieces of their inputs through T_in and lay the parts out in the
// stage.  vec: every block base is 16-byte aligned (bulk copies allowed).
template <int KT>
__device__ __forceinline__ void bd_fill_hdr(const BdMem<KT>& M, BdState* st, const BdTile* __restrict__ desc,
                                            uint32_t total, const uint32_t* __restrict__ dlist,
                                            const uint32_t* __restrict__ first_tile, uint32_t D,
                                            const uint32_t* __restrict__ Tin, bool vec, BdHdr& H) {
  using K = typename KeyTraits<KT>::K;
  constexpr uint32_t VK = 16u / (uint32_t)sizeof(K), VV = 4u;
  const uint32_t lane = threadIdx.x & 31u, P = M.P;
  uint32_t d = 0;
  if (lane == 0) d = atomicAdd(&st->ticket, 1u);
  d = __shfl_sync(0xFFFFFFFFu, d, 0);
  const bool ok = d < D && !*reinterpret_cast<volatile uint32_t*>(&st->err);
  if (!ok) {
    if (lane == 0) H.valid = 0;
    return;
  }
  const uint32_t v = dlist[d];
  const uint32_t tau = first_tile[d] + lane;
  BdTile t{};
  bool in = tau < total;
  if (in) { t = desc[tau]; in = (t.lo >> M.lg) == v; }
  const uint32_t mask = __ballot_sync(0xFFFFFFFFu, in);
  uint32_t nt = __ffs(~mask) ? __ffs(~mask) - 1 : 32u;  // tiles are contiguous
  if (nt > 16) {
    if (lane == 0) atomicExch(&st->err, 2u);  // never: at most 3 pieces when P <= Z
    nt = 16;
  }
  if (lane < nt) H.t[lane] = t;
  __syncwarp();
  // part `lane`: its virtual range, its (at most two) physical pieces, its regions
  uint32_t gq = 0, len = 0;
  if (lane < 2 * nt) {
    const BdTile u = H.t[lane >> 1];
    const uint32_t nA = u.a1 - u.a0;
    if (lane & 1) { gq = u.j + (u.lo - u.i) - u.a0; len = (u.hi - u.lo) - nA; }
    else { gq = u.i + u.a0; len = nA; }
  }
  const uint32_t sk = gq & (VK - 1u), sv = gq & (VV - 1u);
  // region sizes (multiples of the 16-byte unit) and their exclusive prefix
  uint32_t rk = len ? ((sk + len + VK - 1u) / VK + 2u) * VK : 0u;
  uint32_t rv = len ? ((sv + len + VV - 1u) / VV + 2u) * VV : 0u;
  uint32_t ik = rk, iv = rv;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t yk = __shfl_up_sync(0xFFFFFFFFu, ik, o), yv = __shfl_up_sync(0xFFFFFFFFu, iv, o);
    if ((int)lane >= o) { ik += yk; iv += yv; }
  }
  uint32_t slow = 0;
  if (lane < 2 * nt) {
    H.part[lane][0] = gq;
    H.part[lane][1] = len;
    H.ko[lane] = ik - rk + sk;
    H.vo[lane] = iv - rv + sv;
    const uint32_t off = gq & (P - 1), c = min(len, P - off), rest = len - c;
    const uint32_t b1 = len ? Tin[gq >> M.lg] : 0u, b2 = rest ? Tin[(gq + c) >> M.lg] : 0u;
    // the caller's partial last block ends at n: no superset reads there
    const bool bk1 = vec && !(M.has_partial && b1 == M.NB - 1);
    const bool bk2 = vec && !(M.has_partial && b2 == M.NB - 1);
    H.pcb[lane][0] = b1 | (bk1 ? 0u : BD_SLOW);
    H.pcb[lane][1] = b2 | (bk2 ? 0u : BD_SLOW);
    slow = (c && !bk1 ? 1u : 0u) + (rest && !bk2 ? 1u : 0u);
  }
  slow = __reduce_add_sync(0xFFFFFFFFu, slow);
  if (lane == 0) { H.d = d; H.v = v; H.nt = nt; H.nslow = slow; H.valid = 1; }
}

// Warp 0: start the gather of a block's inputs into a stage.  Lane x issues
// part x's bulk copies (keys, then values) after lane 0 has announced the
// block's transaction bytes on `bar`; every thread then copies the pieces
// that cannot go in bulk element by element (cp.async).
template <int KT, bool HV>
__device__ __forceinline__ void bd_issue(const BdMem<KT>& M, const BdHdr& H, typename KeyTraits<KT>::K* sk,
                                         uint32_t* sv, uint64_t* bar) {
  using K = typename KeyTraits<KT>::K;
  constexpr uint32_t VK = 16u / (uint32_t)sizeof(K), VV = 4u;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, P = M.P;
  const uint32_t np = 2 * H.nt;
  if (tid < 32) {
    uint32_t gq = 0, len = 0, c = 0, rest = 0, b1 = 0, b2 = 0, off = 0, sgk = 0, sgv = 0, bytes = 0;
    if (lane < np) {
      gq = H.part[lane][0];
      len = H.part[lane][1];
      off = gq & (P - 1);
      c = min(len, P - off);
      rest = len - c;
      b1 = H.pcb[lane][0];
      b2 = H.pcb[lane][1];
      sgk = gq & (VK - 1u);
      sgv = gq & (VV - 1u);
      if (c && !(b1 & BD_SLOW))
        bytes += ((sgk + c + VK - 1u) / VK) * 16u + (HV ? ((sgv + c + VV - 1u) / VV) * 16u : 0u);
      if (rest && !(b2 & BD_SLOW))
        bytes += ((rest + VK - 1u) / VK) * 16u + (HV ? ((rest + VV - 1u) / VV) * 16u : 0u);
    }
    const uint32_t total = __reduce_add_sync(0xFFFFFFFFu, bytes);
    if (lane == 0) {
      fence_proxy_async_smem();  // this stage's earlier generic reads precede the bulk writes
      mbar_arrive_expect_tx(bar, total);
    }
    __syncwarp();
    if (bytes) {
      const uint32_t ko = H.ko[lane], vo = H.vo[lane];
      if (c && !(b1 & BD_SLOW)) {
        bulk_g2s(sk + ko - sgk, M.kb(b1) + off - sgk, ((sgk + c + VK - 1u) / VK) * 16u, bar);
        if (HV) bulk_g2s(sv + vo - sgv, M.vb(b1) + off - sgv, ((sgv + c + VV - 1u) / VV) * 16u, bar);
      }
      if (rest && !(b2 & BD_SLOW)) {
        bulk_g2s(sk + ko + c, M.kb(b2), ((rest + VK - 1u) / VK) * 16u, bar);
        if (HV) bulk_g2s(sv + vo + c, M.vb(b2), ((rest + VV - 1u) / VV) * 16u, bar);
      }
    }
  }
  if (H.nslow) {  // element-wise pieces (unaligned arrays, the caller's partial last block)
    for (uint32_t x = 0; x < np; ++x) {
      const uint32_t gq = H.part[x][0], len = H.part[x][1], off = gq & (P - 1);
      const uint32_t c = min(len, P - off), rest = len - c;
      const uint32_t b1 = H.pcb[x][0], b2 = H.pcb[x][1];
      if (c && (b1 & BD_SLOW)) {
        const K* gk = M.kb(b1 & ~BD_SLOW) + off;
        for (uint32_t q = tid; q < c; q += BD_THREADS) cp_async_el(sk + H.ko[x] + q, gk + q, (int)sizeof(K));
        if (HV) {
          const uint32_t* gv = M.vb(b1 & ~BD_SLOW) + off;
          for (uint32_t q = tid; q < c; q += BD_THREADS) cp_async_el(sv + H.vo[x] + q, gv + q, 4);
        }
      }
      if (rest && (b2 & BD_SLOW)) {
        const K* gk = M.kb(b2 & ~BD_SLOW);
        for (uint32_t q = tid; q < rest; q += BD_THREADS) cp_async_el(sk + H.ko[x] + c + q, gk + q, (int)sizeof(K));
        if (HV) {
          const uint32_t* gv = M.vb(b2 & ~BD_SLOW);
          for (uint32_t q = tid; q < rest; q += BD_THREADS) cp_async_el(sv + H.vo[x] + c + q, gv + q, 4);
        }
      }
    }
    cp_async_commit();
  }
}

// A stage has landed: its bulk copies (mbarrier phase) and, when the block
// has element-wise pieces, this thread's cp.async groups (the caller then
// synchronises the CTA before anyone reads them).
__device__ __forceinline__ void bd_wait(const BdHdr& H, uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
  if (H.nslow) cp_async_wait_all();
}

// Warp 0: release the input blocks a header's tiles consume (lane x: part x,
// whose <= 2 pieces touch virtual blocks gq / P and gq / P + 1, physical
// blocks from the header).  A block whose counter reaches zero is free; when
// `keep` the first such block is returned to the caller (the CTA's own next
// output block: no trip through the shared ring), the others go to the ring.
// Returns BD_NONE when no block was kept.
__device__ __forceinline__ uint32_t bd_release_hdr(BdState* st, uint32_t* pool, uint32_t cap, uint32_t* remain,
                                                   uint32_t NB, uint32_t P, uint32_t lg, uint32_t has_partial,
                                                   const BdHdr& H, bool keep) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t f0 = BD_NONE, f1 = BD_NONE;
  if (lane < 2 * H.nt) {
    const uint32_t gq = H.part[lane][0], len = H.part[lane][1], off = gq & (P - 1);
    const uint32_t c = min(len, P - off), rest = len - c;
    auto rel = [&](uint32_t v, uint32_t phys, uint32_t cnt) -> uint32_t {
      if (!cnt) return BD_NONE;
      const uint32_t old = atomicSub(&remain[v], cnt);
      if (old != cnt) return BD_NONE;
      if (has_partial && phys == NB - 1) return BD_NONE;  // the partial last block is never freed
      return phys;
    };
    f0 = rel(gq >> lg, H.pcb[lane][0] & ~BD_SLOW, c);
    f1 = rel((gq >> lg) + 1u, H.pcb[lane][1] & ~BD_SLOW, rest);
  }
  const uint32_t m0 = __ballot_sync(0xFFFFFFFFu, f0 != BD_NONE), m1 = __ballot_sync(0xFFFFFFFFu, f1 != BD_NONE);
  // the kept block: the lowest lane's f0, else the lowest lane's f1
  const uint32_t kl = keep ? (m0 ? (uint32_t)__ffs(m0) - 1u : m1 ? (uint32_t)__ffs(m1) - 1u : 32u) : 32u;
  const bool kf0 = m0 != 0u;
  const uint32_t kept = kl < 32u ? __shfl_sync(0xFFFFFFFFu, kf0 ? f0 : f1, kl) : BD_NONE;
  auto push = [&](uint32_t b) {
    const uint32_t at = atomicAdd(&st->tail, 1u);
    reinterpret_cast<volatile uint32_t*>(pool)[at % cap] = b;
  };
  if (f0 != BD_NONE && !(lane == kl && kf0)) push(f0);
  if (f1 != BD_NONE && !(lane == kl && !kf0)) push(f1);
  return kept;
}

// One level pass.  A CTA pipelines two dirty output blocks: while it merges
// block t (inputs in stage t & 1) the inputs of block t+1 stream into the
// other stage (bulk copies on mbarrier t+1 & 1) and warp 1 reads the tiles of
// block t+2.  Before block t takes its output block, block t+1's inputs have
// landed and are released, so whenever every CTA waits for a free block,
// every taken block has released its inputs (no fewer free blocks than an
// in-order round schedule would have).  The merged outputs stay in registers
// and are stored straight into the output block (128-bit stores).  One CTA
// barrier per block (two when the block has element-wise pieces).
template <int KT, bool HV>
__global__ void __launch_bounds__(BD_THREADS) k_bd_level(BdMem<KT> M, BdState* st, const BdTile* __restrict__ desc,
                                                          const uint32_t* __restrict__ info,
                                                          const uint32_t* __restrict__ dlist,
                                                          const uint32_t* __restrict__ first_tile,
                                                          const uint32_t* __restrict__ D_ptr,
                                                          const uint32_t* __restrict__ Tin, uint32_t* __restrict__ Tout,
                                                          uint32_t* __restrict__ pool, uint32_t cap,
                                                          uint32_t* __restrict__ remain) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  constexpr uint32_t OPT = MERGE_K;  // outputs per thread (P <= BD_THREADS * MERGE_K)
  constexpr uint32_t VK = 16u / (uint32_t)sizeof(K);
  extern __shared__ __align__(128) unsigned char bd_smem[];
  const uint32_t P = M.P;
  const uint32_t SEK = bd_stage_elems(P, VK), SEV = bd_stage_elems(P, 4u);
  K* const stk0 = reinterpret_cast<K*>(bd_smem);
  uint32_t* const stv0 = reinterpret_cast<uint32_t*>(stk0 + 2 * SEK);
  auto stk = [&](uint32_t s) { return stk0 + s * SEK; };
  auto stv = [&](uint32_t s) { return stv0 + (HV ? s * SEV : 0u); };
  __shared__ BdHdr hdr[3];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t s_b[2];
  const uint32_t D = *D_ptr, total = info[3];
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  const bool vec = ((reinterpret_cast<uintptr_t>(M.k0) | reinterpret_cast<uintptr_t>(M.v0) |
                     reinterpret_cast<uintptr_t>(M.ks) | reinterpret_cast<uintptr_t>(M.vs)) & 15u) == 0;
  if (blockIdx.x == 0 && tid == 0 && D) atomicAdd(&st->rounds, 1u);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  // prologue: block t = first ticket, gathered and released; header of t+1
  if (warp == 1) bd_fill_hdr<KT>(M, st, desc, total, dlist, first_tile, D, Tin, vec, hdr[0]);
  __syncthreads();
  if (!hdr[0].valid) return;
  bd_issue<KT, HV>(M, hdr[0], stk(0), stv(0), &bar[0]);
  if (warp == 1) bd_fill_hdr<KT>(M, st, desc, total, dlist, first_tile, D, Tin, vec, hdr[1]);
  bd_wait(hdr[0], &bar[0], 0u);
  __syncthreads();
  if (warp == 0) bd_release_hdr(st, pool, cap, remain, M.NB, P, M.lg, M.has_partial, hdr[0], false);
  for (uint32_t it = 0;; ++it) {
    const uint32_t s = it & 1u;
    const BdHdr& H0 = hdr[it % 3];
    BdHdr& H1 = hdr[(it + 1) % 3];
    BdHdr& H2 = hdr[(it + 2) % 3];
    const bool more = H1.valid;
    if (more) bd_issue<KT, HV>(M, H1, stk(s ^ 1u), stv(s ^ 1u), &bar[s ^ 1u]);
    if (warp == 1) {
      if (more) bd_fill_hdr<KT>(M, st, desc, total, dlist, first_tile, D, Tin, vec, H2);
      else if ((tid & 31u) == 0) H2.valid = 0;
    }
    // merge block t into registers: this thread's outputs [OPT tid, OPT tid + OPT)
    const uint32_t v = H0.v, vbase = v << M.lg, len = M.vlen(v), nt = H0.nt;
    const uint32_t c0 = tid * OPT, c1 = min(c0 + OPT, len);
    const K* const sk = stk(s);
    const uint32_t* const sv = stv(s);
    K rk[OPT];
    uint32_t rv[OPT];
    if (nt == 1 && H0.t[0].lo == vbase && H0.t[0].hi == vbase + len && c1 == c0 + OPT) {
      // the block is one merge tile and the chunk is full: branch-free merge
      // over absolute stage indices (a read one past a part stays in its slack)
      const BdTile t = H0.t[0];
      const uint32_t nA = t.a1 - t.a0, nB = len - nA;
      const uint32_t koA = H0.ko[0], koB = H0.ko[1];
      const int32_t dA = (int32_t)H0.vo[0] - (int32_t)koA, dB = (int32_t)H0.vo[1] - (int32_t)koB;
      const uint32_t l = corank<KT>(sk + koA, nA, sk + koB, nB, c0);
      uint32_t ia = koA + l, ib = koB + c0 - l;
      const uint32_t ea = koA + nA, eb = koB + nB;
      K ka = sk[ia], kb = sk[ib];
      typename T::O oa = T::ord(ka), ob = T::ord(kb);
      uint32_t ri[OPT];
#pragma unroll
      for (uint32_t r = 0; r < OPT; ++r) {
        const bool pa = ib >= eb || (ia < ea && oa <= ob);
        rk[r] = pa ? ka : kb;
        ri[r] = pa ? (uint32_t)((int32_t)ia + dA) : (uint32_t)((int32_t)ib + dB);
        ia += pa ? 1u : 0u;
        ib += pa ? 0u : 1u;
        const K nx = sk[pa ? ia : ib];
        const typename T::O onx = T::ord(nx);
        ka = pa ? nx : ka;
        oa = pa ? onx : oa;
        kb = pa ? kb : nx;
        ob = pa ? ob : onx;
      }
      if (HV) {
#pragma unroll
        for (uint32_t r = 0; r < OPT; ++r) rv[r] = sv[ri[r]];
      }
    } else {
      for (uint32_t x = 0; x < nt; ++x) {
        const BdTile t = H0.t[x];
        const uint32_t o = t.lo - vbase, cnt = t.hi - t.lo, nA = t.a1 - t.a0, nB = cnt - nA;
        if (o >= c1 || o + cnt <= c0) continue;
        const uint32_t s0 = max(c0, o) - o;
        const K* A = sk + H0.ko[2 * x];
        const K* B = sk + H0.ko[2 * x + 1];
        const uint32_t* VA = sv + H0.vo[2 * x];
        const uint32_t* VB = sv + H0.vo[2 * x + 1];
        uint32_t ia = corank<KT>(A, nA, B, nB, s0), ib = s0 - ia;
#pragma unroll
        for (uint32_t r = 0; r < OPT; ++r) {
          const uint32_t pos = c0 + r;
          if (pos >= o && pos < o + cnt && pos < c1) {
            const bool takeA = ib >= nB || (ia < nA && T::ord(A[ia]) <= T::ord(B[ib]));
            rk[r] = takeA ? A[ia] : B[ib];
            if (HV) rv[r] = takeA ? VA[ia] : VB[ib];
            ia += takeA ? 1u : 0u;
            ib += takeA ? 0u : 1u;
          }
        }
      }
    }
    if (more) {
      bd_wait(H1, &bar[s ^ 1u], ((it + 1) >> 1) & 1u);  // block t+1's inputs have landed
      if (H1.nslow) __syncthreads();                    // (element-wise pieces: every thread's)
    }
    if (warp == 0) {
      // release block t+1's inputs, then take block t's output block: one the
      // release just freed if any (no ring round trip), else from the ring
      const uint32_t kept =
          more ? bd_release_hdr(st, pool, cap, remain, M.NB, P, M.lg, M.has_partial, H1, true) : BD_NONE;
      if (tid == 0) {
        const uint32_t b = kept != BD_NONE ? kept : bd_alloc(st, pool, cap);
        s_b[s] = b;
        if (b != BD_NONE) Tout[v] = b;
      }
    }
    __syncthreads();  // stage s and header t are no longer read; the output block is known
    const uint32_t b = s_b[s];
    if (b == BD_NONE) break;
    K* dk = M.kb(b);
    uint32_t* dv = HV ? M.vb(b) : nullptr;
    if (vec && c1 == c0 + OPT) {
      store_vec8<K>(dk + c0, rk);
      if (HV) store_vec8<uint32_t>(dv + c0, rv);
    } else {
#pragma unroll
      for (uint32_t r = 0; r < OPT; ++r)
        if (c0 + r < c1) {
          dk[c0 + r] = rk[r];
          if (HV) dv[c0 + r] = rv[r];
        }
    }
    if (!more) break;
  }
}

template <int KT, bool HV>
constexpr size_t bd_level_smem(uint32_t P) {
  return (size_t)2 * bd_stage_elems(P, 16u / (uint32_t)sizeof(typename KeyTraits<KT>::K)) *
             sizeof(typename KeyTraits<KT>::K) +
         (HV ? (size_t)2 * bd_stage_elems(P, 4u) * 4 : 0);
}

// The ring's free blocks into pool[0, count) for the Copy (one CTA).
__global__ void __launch_bounds__(1024) k_bd_ring_to_stack(BdState* st, uint32_t* __restrict__ pool, uint32_t cap,
                                                           uint32_t* __restrict__ tmp) {
  const uint32_t h = st->head, cnt = st->tail - h;
  for (uint32_t x = threadIdx.x; x < cnt; x += blockDim.x) tmp[x] = pool[(h + x) % cap];
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < cnt; x += blockDim.x) pool[x] = tmp[x];
  if (threadIdx.x == 0) st->pool_count = cnt;
}

// After a level: the table maps the dirty blocks to their new homes.
__global__ void k_bd_commit(BdState* st, const uint32_t* __restrict__ dlist, const uint32_t* __restrict__ D_ptr,
                            const uint32_t* __restrict__ Tout, uint32_t* __restrict__ Tin, uint32_t* __restrict__ inv,
                            uint32_t* __restrict__ dirty, uint32_t vb0) {
  const uint32_t D = *D_ptr;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->ticket = 0;  // the next level starts from its first dirty block
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < D; x += gridDim.x * blockDim.x) {
    const uint32_t v = dlist[x], b = Tout[v];
    Tin[v] = b;
    inv[b] = v;  // occupant of b (stale for freed blocks: check Tin[inv[b]] == b)
    dirty[v - vb0] = 0;  // the next pass starts from clean flags
  }
}

// bd_home, step 1: the ring slot holding physical block b, if b is free.
__global__ void k_bd_find_free(const BdState* st, const uint32_t* __restrict__ Tin, const uint32_t* __restrict__ pool,
                               uint32_t cap, uint32_t b, uint32_t* __restrict__ slot) {
  if (Tin[b] == b) return;
  const uint32_t h = st->head, cnt = st->tail - h;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < cnt; x += gridDim.x * blockDim.x)
    if (pool[(h + x) % cap] == b) *slot = (h + x) % cap;
}

// bd_home, step 2 (one CTA): move virtual block b home.  Physical b is free
// (its ring slot now holds b's old location) or holds another virtual block
// u, which moves to a free block first.
template <int KT, bool HV>
__global__ void __launch_bounds__(512) k_bd_home(BdMem<KT> M, BdState* st, uint32_t* __restrict__ Tin,
                                                 uint32_t* __restrict__ inv, uint32_t* __restrict__ pool, uint32_t cap,
                                                 uint32_t b, const uint32_t* __restrict__ slot) {
  using K = typename KeyTraits<KT>::K;
  const uint32_t src = Tin[b];
  if (src == b || st->err) return;
  const uint32_t u = inv[b];
  const bool occupied = u < M.NB && u != b && Tin[u] == b;
  auto copy = [&](uint32_t from, uint32_t to, uint32_t len) {
    const K* sk = M.kb(from);
    K* dk = M.kb(to);
    for (uint32_t q = threadIdx.x; q < len; q += blockDim.x) dk[q] = sk[q];
    if (HV) {
      const uint32_t* sv = M.vb(from);
      uint32_t* dv = M.vb(to);
      for (uint32_t q = threadIdx.x; q < len; q += blockDim.x) dv[q] = sv[q];
    }
  };
  if (occupied) {
    const uint32_t h = st->head;
    if (st->tail == h) { if (threadIdx.x == 0) st->err = 1; return; }
    const uint32_t e = pool[h % cap];
    copy(b, e, M.vlen(u));
    __syncthreads();
    if (threadIdx.x == 0) {
      pool[h % cap] = BD_NONE;
      st->head = h + 1;
      Tin[u] = e;
      inv[e] = u;
    }
  }
  copy(src, b, M.vlen(b));
  __syncthreads();
  if (threadIdx.x == 0) {
    const bool partial_home = M.has_partial && src == M.NB - 1;  // never pooled
    if (!occupied && *slot != 0xFFFFFFFFu) {
      pool[*slot] = partial_home ? BD_NONE : src;  // b's ring slot now offers src
    } else if (!partial_home) {
      const uint32_t t = st->tail;
      pool[t % cap] = src;
      st->tail = t + 1;
    }
    Tin[b] = b;
    inv[b] = b;
  }
}

// --- final Copy: permute blocks into physical order --------------------------
__global__ void k_bd_inverse(const uint32_t* __restrict__ Tin, uint32_t NB, uint32_t nphys,
                             uint32_t* __restrict__ inv) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nphys; b += gridDim.x * blockDim.x) inv[b] = BD_NONE;
}
__global__ void k_bd_inverse2(const uint32_t* __restrict__ Tin, uint32_t NB, uint32_t* __restrict__ inv) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < NB; v += gridDim.x * blockDim.x) inv[Tin[v]] = v;
}

// Final Copy as one cooperative kernel.  Virtual blocks are placed in
// batches [q0, q1) in order (blocks < q0 are home).  For a misplaced block q:
// the later block occupying physical q is evicted into a free block, a source
// inside the batch (another target) is staged into a free block, and then
// every target is written from its source or stage.  CTA 0 plans a batch in
// parallel (its 512 threads, shared memory) while the other CTAs run the
// previous batch's home copies; two grid barriers per batch.  Free blocks
// usable by a batch are pool entries >= q1 (never a target); the batch is
// halved until its evictions + stages fit them.  Sources and stages freed by
// a batch are pooled at plan time: their data is only overwritten by the
// next batch's phase 1, which starts after this batch's phase 2.
constexpr uint32_t BD_CP_THREADS = 512;
constexpr uint32_t BD_CP_BMAX = 1024;   // virtual blocks per batch (2 per planner thread)
constexpr uint32_t BD_CP_PMAX = 4096;   // pool entries the planner looks at (top of the stack)
constexpr uint32_t BD_CP_LIST = 9 * BD_CP_BMAX + 8;  // words per list set: phase 1 (2 B x 3), phase 2 (B x 3), counts

struct BdCopySmem {
  uint32_t src[BD_CP_BMAX], occ[BD_CP_BMAX], need[BD_CP_BMAX], pool[BD_CP_PMAX];
  uint32_t wsum[BD_CP_THREADS / 32];
  uint32_t q0, q1, W, pc, k, total, avail, n2, done;
};

// block-wide exclusive scan of one value per thread (BD_CP_THREADS threads)
__device__ __forceinline__ uint32_t bd_cp_scan(uint32_t v, uint32_t* wsum, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  __syncthreads();
  if (lane == 31) wsum[wp] = x;
  __syncthreads();
  if (wp == 0) {
    uint32_t w = lane < BD_CP_THREADS / 32 ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= (uint32_t)o) w += y;
    }
    if (lane < BD_CP_THREADS / 32) wsum[lane] = w;
  }
  __syncthreads();
  const uint32_t before = wp ? wsum[wp - 1] : 0u;
  *total = wsum[BD_CP_THREADS / 32 - 1];
  return before + x - v;
}

// CTA 0: plan the next batch into list set L (returns with st->copy_q advanced,
// or L[done] = 1 when every block is home).  Layout of L: [0] phase-1 count,
// [1] phase-2 count, [2] done, [8 ...) phase 1 triples (src, dst, len), then
// phase 2 triples at 8 + 6 BMAX.
__device__ void bd_copy_plan_cta(BdState* st, uint32_t* __restrict__ Tin, uint32_t* __restrict__ inv,
                                 uint32_t* __restrict__ pool, uint32_t NB, uint32_t P, uint32_t n,
                                 uint32_t has_partial, uint32_t* __restrict__ L, BdCopySmem& S) {
  const uint32_t tid = threadIdx.x;
  auto vlen = [&](uint32_t v) -> uint32_t { return v + 1 < NB ? P : n - v * P; };
  if (tid == 0) {
    uint32_t q0 = st->copy_q;
    S.q0 = q0;
    S.W = st->err ? 0u : min(BD_CP_BMAX, NB - q0);
    S.pc = st->pool_count;
    S.k = min(S.pc, BD_CP_PMAX);
  }
  __syncthreads();
  const uint32_t q0 = S.q0, W = S.W, pc = S.pc, k = S.k;
  if (W == 0) {
    if (tid == 0) { L[0] = L[1] = 0; L[2] = 1; }
    return;
  }
  for (uint32_t x = tid; x < W; x += BD_CP_THREADS) {
    S.src[x] = Tin[q0 + x];
    S.occ[x] = inv[q0 + x];
  }
  for (uint32_t y = tid; y < k; y += BD_CP_THREADS) S.pool[y] = pool[pc - k + y];  // top of the stack
  __syncthreads();
  // the largest batch (halving from W) whose evictions + stages fit the free
  // blocks >= q1
  uint32_t q1 = q0 + W;
  uint32_t total = 0, avail = 0;
  for (;;) {
    uint32_t mine = 0;
    for (uint32_t x = 2 * tid; x < 2 * tid + 2; ++x) {
      uint32_t nd = 0;
      if (x < q1 - q0) {
        const uint32_t q = q0 + x, src = S.src[x], occ = S.occ[x];
        if (src != q) nd = (occ != BD_NONE && occ >= q1 ? 1u : 0u) + (src < q1 ? 1u : 0u);
      }
      S.need[x] = nd;
      mine += nd;
    }
    uint32_t t0;
    bd_cp_scan(mine, S.wsum, &t0);
    uint32_t av = 0;
    for (uint32_t y = tid; y < k; y += BD_CP_THREADS) av += S.pool[y] >= q1 ? 1u : 0u;
    uint32_t a0;
    bd_cp_scan(av, S.wsum, &a0);
    total = t0;
    avail = a0;
    if (total <= avail || q1 == q0 + 1) break;
    q1 = q0 + max(1u, (q1 - q0) / 2);
  }
  if (total > avail) {  // even one block does not fit
    if (tid == 0) {
      if (k == pc) st->err = 1;
      else {  // drop the dead (< q1) entries of the window and retry next time
        uint32_t o = pc - k;
        for (uint32_t y = 0; y < k; ++y) if (S.pool[y] >= q1) pool[o++] = S.pool[y];
        st->pool_count = o;
      }
      L[0] = L[1] = 0; L[2] = st->err;
    }
    return;
  }
  // free list: the window's entries >= q1, compacted to S.pool[0, avail)
  uint32_t vals[BD_CP_PMAX / BD_CP_THREADS];
  uint32_t nm = 0;
  for (uint32_t y = tid; y < k; y += BD_CP_THREADS)
    if (S.pool[y] >= q1) vals[nm++] = S.pool[y];
  uint32_t tot;
  const uint32_t fo = bd_cp_scan(nm, S.wsum, &tot);
  __syncthreads();
  for (uint32_t z = 0; z < nm; ++z) S.pool[fo + z] = vals[z];
  __syncthreads();
  // assignments
  uint32_t nd2[2], mis[2], mine = 0, mcount = 0;
  for (uint32_t u = 0; u < 2; ++u) {
    const uint32_t x = 2 * tid + u;
    nd2[u] = x < q1 - q0 ? S.need[x] : 0u;
    mis[u] = (x < q1 - q0 && S.src[x] != q0 + x) ? 1u : 0u;
    mine += nd2[u];
    mcount += mis[u];
  }
  uint32_t t1, t2;
  uint32_t off = bd_cp_scan(mine, S.wsum, &t1);
  uint32_t off2 = bd_cp_scan(mcount, S.wsum, &t2);
  // freed blocks (direct sources outside the batch, stages) go after the
  // unused free entries: count them
  uint32_t fr = 0;
  for (uint32_t u = 0; u < 2; ++u) {
    const uint32_t x = 2 * tid + u;
    if (!mis[u]) continue;
    const uint32_t src = S.src[x];
    const bool stg = src < q1;
    if (stg) ++fr;                                              // the stage block
    else if (!(has_partial && src == NB - 1)) ++fr;              // the old home of q
  }
  uint32_t tf;
  uint32_t offf = bd_cp_scan(fr, S.wsum, &tf);
  uint32_t* L1 = L + 8;
  uint32_t* L2 = L + 8 + 6 * BD_CP_BMAX;
  const uint32_t base_new = pc - k + (avail - total);  // pool: [0, pc-k) untouched, unused entries, freed
  for (uint32_t u = 0; u < 2; ++u) {
    const uint32_t x = 2 * tid + u;
    if (!mis[u]) continue;
    const uint32_t q = q0 + x, src = S.src[x], occ = S.occ[x];
    const bool ev = occ != BD_NONE && occ >= q1, stg = src < q1;
    uint32_t o = off;
    if (ev) {
      const uint32_t e = S.pool[o];
      L1[3 * o] = q; L1[3 * o + 1] = e; L1[3 * o + 2] = vlen(occ);
      Tin[occ] = e;
      inv[e] = occ;
      ++o;
    }
    uint32_t from = src;
    if (stg) {
      const uint32_t t = S.pool[o];
      L1[3 * o] = src; L1[3 * o + 1] = t; L1[3 * o + 2] = vlen(q);
      from = t;
      ++o;
      pool[base_new + offf++] = t;
    } else {
      inv[src] = BD_NONE;
      if (!(has_partial && src == NB - 1)) pool[base_new + offf++] = src;
    }
    off = o;
    L2[3 * off2] = from; L2[3 * off2 + 1] = q; L2[3 * off2 + 2] = vlen(q);
    ++off2;
    Tin[q] = q;
  }
  __syncthreads();
  // inv of the targets last: a stage source src < q1 is itself a target of
  // this batch (inv[src] = src set by its own thread)
  for (uint32_t u = 0; u < 2; ++u) {
    const uint32_t x = 2 * tid + u;
    if (mis[u]) inv[q0 + x] = q0 + x;
  }
  // unused free entries of the window
  for (uint32_t y = total + tid; y < avail; y += BD_CP_THREADS) pool[pc - k + (y - total)] = S.pool[y];
  __syncthreads();
  if (tid == 0) {
    st->pool_count = base_new + tf;
    st->copy_q = q1;
    st->copies += t1 + t2;
    L[0] = t1;
    L[1] = t2;
    L[2] = 0;
  }
}

template <int KT, bool HV>
__device__ __forceinline__ void bd_copy_list(const BdMem<KT>& M, const uint32_t* __restrict__ list, uint32_t cnt,
                                             uint32_t first, uint32_t stride) {
  using K = typename KeyTraits<KT>::K;
  // 16-byte vectors when every block base is aligned (the caller's array may
  // start anywhere: sub-arrays of the dyadic-cell mode)
  const bool vec = ((reinterpret_cast<uintptr_t>(M.k0) | reinterpret_cast<uintptr_t>(M.v0) |
                     reinterpret_cast<uintptr_t>(M.ks) | reinterpret_cast<uintptr_t>(M.vs)) & 15u) == 0;
  for (uint32_t c = first; c < cnt; c += stride) {
    const uint32_t a = list[3 * c], b = list[3 * c + 1], len = list[3 * c + 2];
    const K* sk = M.kb(a);
    K* dk = M.kb(b);
    constexpr uint32_t KV = 16 / sizeof(K);
    const uint32_t nv = vec ? len / KV : 0u;
    for (uint32_t q = threadIdx.x; q < nv; q += blockDim.x)
      reinterpret_cast<uint4*>(dk)[q] = __ldcg(reinterpret_cast<const uint4*>(sk) + q);
    for (uint32_t q = nv * KV + threadIdx.x; q < len; q += blockDim.x) dk[q] = sk[q];
    if (HV) {
      const uint32_t* sv = M.vb(a);
      uint32_t* dv = M.vb(b);
      const uint32_t nv4 = vec ? len / 4 : 0u;
      for (uint32_t q = threadIdx.x; q < nv4; q += blockDim.x)
        reinterpret_cast<uint4*>(dv)[q] = __ldcg(reinterpret_cast<const uint4*>(sv) + q);
      for (uint32_t q = nv4 * 4 + threadIdx.x; q < len; q += blockDim.x) dv[q] = sv[q];
    }
  }
}

// The whole Copy (cooperative launch, gridDim.x >= 2).  lists: 2 list sets of
// BD_CP_LIST words.
template <int KT, bool HV>
__global__ void __launch_bounds__(BD_CP_THREADS) k_bd_copy_all(BdMem<KT> M, BdState* st, uint32_t* Tin, uint32_t* inv,
                                                                uint32_t* pool, uint32_t* lists) {
  __shared__ BdCopySmem S;
  cg::grid_group grid = cg::this_grid();
  uint32_t j = 0;
  if (blockIdx.x == 0) bd_copy_plan_cta(st, Tin, inv, pool, M.NB, M.P, M.n, M.has_partial, lists, S);
  grid.sync();
  for (;;) {
    uint32_t* L = lists + (size_t)(j & 1) * BD_CP_LIST;
    const uint32_t n1 = ((volatile uint32_t*)L)[0], n2 = ((volatile uint32_t*)L)[1],
                   done = ((volatile uint32_t*)L)[2];
    if (done) break;
    bd_copy_list<KT, HV>(M, L + 8, n1, blockIdx.x, gridDim.x);  // phase 1: evictions and stages
    grid.sync();
    if (blockIdx.x == 0)
      bd_copy_plan_cta(st, Tin, inv, pool, M.NB, M.P, M.n, M.has_partial, lists + (size_t)((j + 1) & 1) * BD_CP_LIST, S);
    else
      bd_copy_list<KT, HV>(M, L + 8 + 6 * BD_CP_BMAX, n2, blockIdx.x - 1, gridDim.x - 1);  // phase 2: targets
    grid.sync();
    ++j;
  }
}

// Initial pool: the scratch blocks.
// Initial ring: the scratch blocks, every other slot empty.
__global__ void k_bd_init(BdState* st, uint32_t* __restrict__ pool, uint32_t cap, uint32_t* __restrict__ Tin,
                          uint32_t* __restrict__ inv, uint32_t NB, uint32_t F, uint32_t* __restrict__ dirty) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < NB; v += gridDim.x * blockDim.x) Tin[v] = v;
  // dirty flags start (and, cleared by every commit, stay) zero
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < NB + 8; v += gridDim.x * blockDim.x) dirty[v] = 0;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < cap; x += gridDim.x * blockDim.x) {
    pool[x] = x < F ? NB + x : BD_NONE;
    inv[x] = x < NB ? x : BD_NONE;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->head = 0; st->tail = F; st->ticket = 0; st->err = 0; st->pool_count = 0;
    st->rounds = 0; st->copies = 0; st->copy_q = 0;
  }
}

}  // namespace vmps
