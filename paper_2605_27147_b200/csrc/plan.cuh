// plan.cuh -- node powers, the Powersort merge tree and its level schedule.
//
// Boundary t (1 <= t < r) sits between runs t-1 = [i,j) and t = [j,k).
// Power: least p with floor(a 2^p) != floor(b 2^p) for
// a = (i+j)/2n, b = (j+k)/2n, found by bisecting both binary expansions with
// exact integer arithmetic (a different derivation from the oracle's).
// Alg. 1's merge tree is the Cartesian tree of the powers (min at the root):
// node t's segment is the maximal run interval around t whose inner
// boundaries all have power >= p_t.  Those runs are exactly the runs whose
// midpoint lies in t's dyadic cell of level q = p_t - 1, i.e.
// floor((s_u + s_{u+1}) 2^q / 2n) == c, where c = floor(a 2^q) is the common
// prefix of a and b -- found by galloping over the sorted run midpoints.
// Depth (ping-pong parity) and the count of left
// ancestors (Alg. 1's post-order rank) come from pointer jumping.
#pragma once
#include "vmps_internal.cuh"

namespace vmps {

typedef unsigned __int128 u128;

__device__ __forceinline__ uint32_t node_power(uint64_t n, uint64_t i, uint64_t j, uint64_t k,
                                               uint64_t* prefix) {
  uint64_t A = i + j, B = j + k, N2 = 2 * n, c = 0;
  uint32_t p = 0;
  for (;;) {
    ++p;
    A <<= 1;
    B <<= 1;
    bool ba = A >= N2, bb = B >= N2;
    if (ba != bb) break;
    if (ba) { A -= N2; B -= N2; }
    c = (c << 1) | (uint64_t)ba;
  }
  *prefix = c;
  return p;
}

// K5 + K6: powers and segments.
template <typename P>
__global__ void k_powers_seg(const P* __restrict__ rs, uint64_t n, const uint32_t* scalars,
                             uint8_t* __restrict__ power, uint32_t* __restrict__ seg_l,
                             uint32_t* __restrict__ seg_r) {
  const uint32_t r = scalars[SC_RUNS];
  const bool pow2 = (n & (n - 1)) == 0;
  const uint32_t L2n = 64u - (uint32_t)__clzll((long long)(2 * n)) - 1u;  // log2(2n) when pow2
  for (uint32_t t = 1 + blockIdx.x * blockDim.x + threadIdx.x; t < r;
       t += gridDim.x * blockDim.x) {
    uint64_t c, lo_thr, hi_thr;
    uint32_t p;
    if (pow2) {
      // 2n = 2^L: a = A / 2^L exactly, so floor(a 2^p) = A >> (L - p) and the
      // least p where A and B differ is L - h, h = the highest bit of A ^ B;
      // the common prefix c = A >> (h + 1) and 2n / 2^q = 2^(h+1) (q = p - 1)
      const uint64_t A = (uint64_t)rs[t - 1] + rs[t], B = (uint64_t)rs[t] + rs[t + 1];
      const uint32_t h = 63u - (uint32_t)__clzll((long long)(A ^ B));
      p = L2n - h;
      c = A >> (h + 1);
      lo_thr = c << (h + 1);
      hi_thr = (c + 1) << (h + 1);
    } else {
      p = node_power(n, rs[t - 1], rs[t], rs[t + 1], &c);
      const uint32_t q = p - 1;
      // s_u 2^q >= c 2n  <=>  s_u >= ceil(c 2n / 2^q), with s_u = rs[u] + rs[u+1]
      // (both thresholds < 2^34: c < 2^q); the loops compare 64-bit sums only
      const u128 N2 = (u128)(2ull * n);
      const u128 one = 1;
      lo_thr = (uint64_t)(((u128)c * N2 + (one << q) - 1) >> q);
      hi_thr = (uint64_t)(((u128)(c + 1) * N2 + (one << q) - 1) >> q);
    }
    power[t] = (uint8_t)p;
    auto mid_scaled = [&](uint32_t u) -> uint64_t { return (uint64_t)rs[u] + (uint64_t)rs[u + 1]; };
    // L = smallest u in [0, t-1] with mid(u) 2^q >= c 2n (run t-1 qualifies)
    int64_t good = (int64_t)t - 1, bad = -1;
    for (int64_t step = 1;; step <<= 1) {
      int64_t u = good - step;
      if (u < 0) { if (mid_scaled(0) >= lo_thr) { good = 0; } else { bad = 0; } break; }
      if (mid_scaled((uint32_t)u) >= lo_thr) good = u;
      else { bad = u; break; }
    }
    while (good - bad > 1) {
      int64_t m = bad + (good - bad) / 2;
      if (mid_scaled((uint32_t)m) >= lo_thr) good = m; else bad = m;
    }
    seg_l[t] = (uint32_t)good;
    // R = largest u in [t, r-1] with mid(u) 2^q < (c+1) 2n (run t qualifies)
    int64_t g2 = t, b2 = r;
    for (int64_t step = 1;; step <<= 1) {
      int64_t u = g2 + step;
      if (u > (int64_t)r - 1) {
        if (mid_scaled(r - 1) < hi_thr) g2 = r - 1; else b2 = r - 1;
        break;
      }
      if (mid_scaled((uint32_t)u) < hi_thr) g2 = u;
      else { b2 = u; break; }
    }
    while (b2 - g2 > 1) {
      int64_t m = g2 + (b2 - g2) / 2;
      if (mid_scaled((uint32_t)m) < hi_thr) g2 = m; else b2 = m;
    }
    seg_r[t] = (uint32_t)g2 + 1;
  }
}

// Parent = the neighbouring smaller-power boundary with the larger power;
// initialise pointer jumping: dep = depth (low 16) | left-ancestors (high 16).
__global__ void k_parent_init(const uint32_t* scalars, const uint8_t* __restrict__ power,
                              const uint32_t* __restrict__ seg_l,
                              const uint32_t* __restrict__ seg_r, uint32_t* __restrict__ parent,
                              uint32_t* __restrict__ anc, uint32_t* __restrict__ dep) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t t = 1 + blockIdx.x * blockDim.x + threadIdx.x; t < r;
       t += gridDim.x * blockDim.x) {
    uint32_t a = seg_l[t], b = seg_r[t];  // boundary a (if >= 1), boundary b (if < r)
    uint32_t par = 0;
    bool ha = a >= 1, hb = b < r;
    if (ha && hb) par = power[a] > power[b] ? a : b;
    else if (ha) par = a;
    else if (hb) par = b;
    parent[t] = par;
    anc[t] = par;
    dep[t] = par ? (1u | ((par < t) ? (1u << 16) : 0u)) : 0u;
  }
}

__global__ void k_jump(const uint32_t* scalars, const uint32_t* __restrict__ anc_in,
                       const uint32_t* __restrict__ dep_in, uint32_t* __restrict__ anc_out,
                       uint32_t* __restrict__ dep_out) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t t = 1 + blockIdx.x * blockDim.x + threadIdx.x; t < r;
       t += gridDim.x * blockDim.x) {
    uint32_t a = anc_in[t];
    if (a) {
      anc_out[t] = anc_in[a];
      dep_out[t] = dep_in[t] + dep_in[a];
    } else {
      anc_out[t] = 0;
      dep_out[t] = dep_in[t];
    }
  }
}

// Buffer of an item (node output, unit or leaf) at tree depth t: depth parity
// for level-by-level merges; with two-level merges (only even depths
// materialized) the item consumed by its nearest even-depth ancestor.
__device__ __forceinline__ uint32_t item_buf(uint32_t t, int fuse2) {
  if (!fuse2) return t & 1u;
  return (t & 1u) ? (1u - (((t - 1u) >> 1) & 1u)) : ((t >> 1) & 1u);
}

__device__ __forceinline__ uint32_t seg_size(const uint32_t* rs, const uint32_t* seg_l,
                                             const uint32_t* seg_r, uint32_t t) {
  return rs[seg_r[t]] - rs[seg_l[t]];
}

// Node classification: fused unit roots, non-fused nodes (level histogram),
// merge cost M.
__global__ void k_class_nodes(const uint32_t* __restrict__ rs, uint32_t* scalars,
                              unsigned long long* counters, const uint8_t* __restrict__ power,
                              const uint32_t* __restrict__ seg_l, const uint32_t* __restrict__ seg_r,
                              const uint32_t* __restrict__ parent, const uint32_t* __restrict__ dep,
                              uint32_t fuse_z, uint32_t* __restrict__ unit_end,
                              uint8_t* __restrict__ unit_par, uint32_t* __restrict__ level_cnt, int fuse2) {
  const uint32_t r = scalars[SC_RUNS];
  unsigned long long m = 0, fm = 0, hm = 0;  // M, fused M, elements of HBM merge passes
  uint32_t maxp = 0;
  for (uint32_t t = 1 + blockIdx.x * blockDim.x + threadIdx.x; t < r;
       t += gridDim.x * blockDim.x) {
    uint32_t size = seg_size(rs, seg_l, seg_r, t);
    m += size;
    uint32_t p = power[t];
    maxp = max(maxp, p);
    if (size <= fuse_z) {
      fm += size;
      uint32_t par = parent[t];
      uint32_t psize = par ? seg_size(rs, seg_l, seg_r, par) : 0xFFFFFFFFu;
      if (psize > fuse_z) {
        uint32_t u = seg_l[t];
        unit_end[u] = rs[seg_r[t]];
        unit_par[u] = (uint8_t)item_buf(dep[t] & 0xFFFFu, fuse2);
      }
    } else if (!fuse2 || (dep[t] & 1u) == 0) {  // two-level mode: only even depths are materialized
      atomicAdd(&level_cnt[p], 1u);
      hm += size;
    }
  }
  // warp-aggregate the counters
  for (int o = 16; o; o >>= 1) {
    m += __shfl_xor_sync(0xFFFFFFFFu, m, o);
    fm += __shfl_xor_sync(0xFFFFFFFFu, fm, o);
    hm += __shfl_xor_sync(0xFFFFFFFFu, hm, o);
    maxp = max(maxp, __shfl_xor_sync(0xFFFFFFFFu, maxp, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (m) atomicAdd(&counters[0], m);
    if (fm) atomicAdd(&counters[1], fm);
    if (hm) atomicAdd(&counters[2], hm);
    if (maxp) atomicMax(&scalars[SC_MAXPOW], maxp);
  }
}

// Leaf classification: unit starts (and leaf-rooted units), long leaves.
// Also zero-fills flags in [r, cap] so the scans see a clean tail.
__global__ void k_class_runs(const uint32_t* __restrict__ rs, const uint8_t* __restrict__ kind,
                             const uint32_t* scalars, const uint8_t* __restrict__ power,
                             const uint32_t* __restrict__ seg_l, const uint32_t* __restrict__ seg_r,
                             const uint32_t* __restrict__ dep, uint32_t fuse_z, uint32_t cap,
                             uint32_t* __restrict__ unit_flag, uint32_t* __restrict__ long_flag,
                             uint32_t* __restrict__ unit_end, uint8_t* __restrict__ unit_par,
                             uint8_t* __restrict__ long_par, int fuse2) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u <= cap;
       u += gridDim.x * blockDim.x) {
    if (u >= r) {
      unit_flag[u] = 0;
      long_flag[u] = 0;
      continue;
    }
    uint32_t size = rs[u + 1] - rs[u];
    // parent of leaf u: boundary u or u+1, the one with the larger power
    uint32_t pl = 0;
    bool ha = u >= 1, hb = u + 1 < r;
    if (ha && hb) pl = power[u] > power[u + 1] ? u : u + 1;
    else if (ha) pl = u;
    else if (hb) pl = u + 1;
    uint32_t dleaf = pl ? (dep[pl] & 0xFFFFu) + 1u : 0u;
    if (size > fuse_z) {
      long_flag[u] = 1;
      unit_flag[u] = 0;
      long_par[u] = (uint8_t)(item_buf(dleaf, fuse2) | ((kind[u] & VMPS_RUN_DESC) ? 2u : 0u));
    } else {
      long_flag[u] = 0;
      bool start = (u == 0) || seg_size(rs, seg_l, seg_r, u) > fuse_z;
      unit_flag[u] = start ? 1u : 0u;
      if (start) {
        bool leaf_root = (pl == 0) || seg_size(rs, seg_l, seg_r, pl) > fuse_z;
        if (leaf_root) {
          unit_end[u] = rs[u + 1];
          unit_par[u] = (uint8_t)item_buf(dleaf, fuse2);
        }
      }
    }
  }
}

constexpr uint32_t LONG_CHUNK = 4096;

// Compact units (start, end, parity) and long leaves (start, end, flags,
// chunk count) in position order.
__global__ void k_compact(const uint32_t* __restrict__ rs, uint32_t* scalars,
                          const uint32_t* __restrict__ unit_flag,
                          const uint32_t* __restrict__ unit_idx,
                          const uint32_t* __restrict__ long_flag,
                          const uint32_t* __restrict__ long_idx,
                          const uint32_t* __restrict__ unit_end, const uint8_t* __restrict__ unit_par,
                          const uint8_t* __restrict__ long_par, uint32_t* __restrict__ units,
                          uint32_t* __restrict__ longs, uint32_t* __restrict__ long_chunks,
                          uint32_t par_mask) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u <= r;
       u += gridDim.x * blockDim.x) {
    if (u == r) {
      scalars[SC_UNITS] = unit_idx[r];
      scalars[SC_LONG] = long_idx[r];
      long_chunks[long_idx[r]] = 0;
      continue;
    }
    if (unit_flag[u]) {
      uint32_t x = unit_idx[u];
      units[3 * x + 0] = rs[u];
      units[3 * x + 1] = unit_end[u];
      units[3 * x + 2] = unit_par[u] & par_mask;
    }
    if (long_flag[u]) {
      uint32_t x = long_idx[u];
      uint32_t s = rs[u], e = rs[u + 1], f = long_par[u] & (2u | par_mask);
      longs[4 * x + 0] = s;
      longs[4 * x + 1] = e;
      longs[4 * x + 2] = f;
      bool desc = f & 2u, odd = f & 1u;
      uint32_t work = desc ? (odd ? e - s : (e - s) / 2) : (odd ? e - s : 0u);
      long_chunks[x] = (work + LONG_CHUNK - 1) / LONG_CHUNK;
    }
  }
}

// Level bucketing of non-fused nodes by power (ascending), one block.
__global__ void k_level_scan(uint32_t* level_cnt, uint32_t* level_start, uint32_t* scalars) {
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int p = 0; p < LEVEL_SLOTS; ++p) {
      level_start[p] = acc;
      acc += level_cnt[p];
    }
    level_start[LEVEL_SLOTS] = acc;
    scalars[SC_NONFUSED] = acc;
  }
}

__global__ void k_level_scatter(const uint32_t* __restrict__ rs, const uint32_t* scalars,
                                const uint8_t* __restrict__ power,
                                const uint32_t* __restrict__ seg_l,
                                const uint32_t* __restrict__ seg_r, uint32_t fuse_z,
                                const uint32_t* __restrict__ level_start,
                                uint32_t* __restrict__ level_fill, uint32_t* __restrict__ lnodes,
                                const uint32_t* __restrict__ dep, int fuse2) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t t = 1 + blockIdx.x * blockDim.x + threadIdx.x; t < r;
       t += gridDim.x * blockDim.x) {
    if (seg_size(rs, seg_l, seg_r, t) > fuse_z && (!fuse2 || (dep[t] & 1u) == 0)) {
      uint32_t p = power[t];
      uint32_t pos = level_start[p] + atomicAdd(&level_fill[p], 1u);
      lnodes[pos] = t;
    }
  }
}

// Tiles per bucketed node (zero-filled tail up to cap).
__global__ void k_level_tiles(const uint32_t* __restrict__ rs, const uint32_t* scalars,
                              const uint32_t* __restrict__ seg_l, const uint32_t* __restrict__ seg_r,
                              const uint32_t* __restrict__ lnodes, uint32_t tout, uint32_t cap,
                              uint32_t* __restrict__ tiles) {
  const uint32_t m = scalars[SC_NONFUSED];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= cap;
       x += gridDim.x * blockDim.x) {
    uint32_t c = 0;
    if (x < m) {  // tiles aligned to global multiples of tout (see k_tile_desc)
      uint32_t t = lnodes[x];
      uint32_t i = rs[seg_l[t]], k = rs[seg_r[t]];
      c = (k + tout - 1) / tout - i / tout;
    }
    tiles[x] = c;
  }
}

__global__ void k_level_tile_off(const uint32_t* __restrict__ level_start,
                                 const uint32_t* __restrict__ ltiles, uint32_t* level_tile) {
  int p = threadIdx.x;
  if (p <= LEVEL_SLOTS) level_tile[p] = ltiles[level_start[p]];
}

// Post-order rank of node t in Alg. 1's execution order: merges run in
// increasing (trigger, -t) with trigger = next smaller boundary = seg_r[t];
// this is the post-order of the Cartesian tree, whose rank is
// (seg_r[t] - 1) - (left ancestors of t) - 1.
template <typename P>
__global__ void k_plan_records(const P* __restrict__ rs, const uint32_t* scalars,
                               const uint8_t* __restrict__ power, const uint32_t* __restrict__ seg_l,
                               const uint32_t* __restrict__ seg_r, const uint32_t* __restrict__ dep,
                               const uint8_t* __restrict__ kind, uint64_t* __restrict__ run_start,
                               uint8_t* __restrict__ run_kind, vmps_merge_rec_t* __restrict__ merges) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < r;
       t += gridDim.x * blockDim.x) {
    run_start[t] = rs[t];
    run_kind[t] = kind[t];
    if (t == 0) continue;
    uint32_t la = dep[t] >> 16;
    uint32_t ord = seg_r[t] - 2 - la;
    vmps_merge_rec_t rec;
    rec.i = rs[seg_l[t]];
    rec.j = rs[t];
    rec.k = rs[seg_r[t]];
    rec.power = power[t];
    rec.order = ord;
    merges[ord] = rec;
  }
}

// Merge records only (the distributed plan supplies its own run arrays).
template <typename P>
__global__ void k_plan_records_only(const P* __restrict__ rs, const uint32_t* scalars,
                                    const uint8_t* __restrict__ power, const uint32_t* __restrict__ seg_l,
                                    const uint32_t* __restrict__ seg_r, const uint32_t* __restrict__ dep,
                                    vmps_merge_rec_t* __restrict__ merges) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t t = 1 + blockIdx.x * blockDim.x + threadIdx.x; t < r; t += gridDim.x * blockDim.x) {
    const uint32_t ord = seg_r[t] - 2 - (dep[t] >> 16);
    vmps_merge_rec_t rec;
    rec.i = rs[seg_l[t]];
    rec.j = rs[t];
    rec.k = rs[seg_r[t]];
    rec.power = power[t];
    rec.order = ord;
    merges[ord] = rec;
  }
}

// Zero arr[x] for x in [scalars[which], cap] (clean tail before a scan).
__global__ void k_zero_tail(uint32_t* __restrict__ arr, const uint32_t* scalars, int which, uint32_t cap) {
  const uint32_t from = scalars[which];
  for (uint32_t x = from + blockIdx.x * blockDim.x + threadIdx.x; x <= cap; x += gridDim.x * blockDim.x)
    arr[x] = 0;
}

// Every non-fused node must lie on a launched level (p <= p_hi), and (4-way
// schedule) no level may have had more tiles than the descriptor array holds
// (the bound in carve() is exact; checked after the fact so the hot kernels
// carry no extra test).
__global__ void k_check_levels(const uint32_t* level_cnt, int p_hi, uint32_t* scalars,
                               const uint32_t* level_tile, uint32_t tile_cap) {
  for (int p = p_hi + 1 + threadIdx.x; p < LEVEL_SLOTS; p += blockDim.x)
    if (level_cnt[p]) scalars[SC_ERROR] = 1;
  if (level_tile)
    for (int p = 1 + threadIdx.x; p <= p_hi; p += blockDim.x)
      if (level_tile[p + 1] - level_tile[p] > tile_cap) scalars[SC_ERROR] = 2;
}

// Internal-consistency guard of a sort called without h_stats (nothing is
// read back to report VMPS_ERR_INTERNAL): a tripped SC_ERROR aborts the
// kernel, so the error surfaces loudly at the caller's next synchronisation
// instead of a silently partial result.  Never expected to fire.
__global__ void k_error_guard(const uint32_t* scalars) {
  if (scalars[SC_ERROR]) __trap();
}

// ---------------------------------------------------------------------------
// Exclusive scan of u32 (block scan + recursive block offsets).
// ---------------------------------------------------------------------------
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tiles(const uint32_t* __restrict__ in,
                                                             uint32_t* __restrict__ out, uint32_t len,
                                                             uint32_t* __restrict__ bsum) {
  __shared__ uint32_t wsum[SCAN_THREADS / 32];
  const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  uint32_t v[SCAN_ITEMS], s = 0;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    v[q] = base + q < len ? in[base + q] : 0u;
    s += v[q];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < SCAN_THREADS / 32 ? wsum[lane] : 0u;
    uint32_t wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < SCAN_THREADS / 32) wsum[lane] = wi - w;
    if (lane == SCAN_THREADS / 32 - 1) bsum[blockIdx.x] = wi;
  }
  __syncthreads();
  uint32_t run = wsum[warp] + incl - s;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    if (base + q < len) out[base + q] = run;
    run += v[q];
  }
}

__global__ void k_scan_add(uint32_t* __restrict__ out, uint32_t len, const uint32_t* __restrict__ boff) {
  const uint32_t base = blockIdx.x * SCAN_TILE;
  const uint32_t add = boff[blockIdx.x];
  for (uint32_t q = threadIdx.x; q < SCAN_TILE; q += blockDim.x)
    if (base + q < len) out[base + q] += add;
}


// Single-pass exclusive scan (decoupled look-back): a CTA scans its tile of
// SCAN1_TILE values (128-bit loads / stores), publishes its aggregate, then
// warp 0 sums its predecessors' published values 32 at a time until it meets
// an inclusive prefix, and publishes its own.  Status word per tile:
// bit 32 = aggregate, bit 33 = inclusive prefix, low 32 bits the value
// (zeroed before the launch).  A CTA waits only on lower-numbered tiles,
// which are dispatched before it.  One read and one write of the array,
// against four passes and a recursion for k_scan_tiles / k_scan_add.
constexpr int SCAN1_THREADS = 256;
constexpr int SCAN1_ITEMS = 16;
constexpr int SCAN1_TILE = SCAN1_THREADS * SCAN1_ITEMS;

__global__ void __launch_bounds__(SCAN1_THREADS) k_scan1(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                         uint32_t len, unsigned long long* status) {
  __shared__ uint32_t wsum[SCAN1_THREADS / 32];
  __shared__ uint32_t s_prefix;
  const uint32_t tile = blockIdx.x;
  const uint32_t base = tile * SCAN1_TILE + threadIdx.x * SCAN1_ITEMS;
  const bool vec = base + SCAN1_ITEMS <= len && ((((uintptr_t)in) | ((uintptr_t)out)) & 15u) == 0;
  uint32_t v[SCAN1_ITEMS], s = 0;
  if (vec) {
    const uint4* src = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
    for (int q = 0; q < SCAN1_ITEMS / 4; ++q) {
      const uint4 x = src[q];
      v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < SCAN1_ITEMS; ++q) v[q] = base + q < len ? in[base + q] : 0u;
  }
#pragma unroll
  for (int q = 0; q < SCAN1_ITEMS; ++q) s += v[q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < SCAN1_THREADS / 32 ? wsum[lane] : 0u;
    uint32_t wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < SCAN1_THREADS / 32) wsum[lane] = wi - w;
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, wi, SCAN1_THREADS / 32 - 1);
    volatile unsigned long long* st = status;
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = (2ull << 32) | total;
    } else {
      if (lane == 0) st[tile] = (1ull << 32) | total;
      for (int32_t j = (int32_t)tile - 1 - lane;; j -= 32) {
        unsigned long long x = 2ull << 32;  // before tile 0: an empty inclusive prefix
        if (j >= 0)
          do { x = st[j]; } while ((x >> 32) == 0);
        const uint32_t isp = __ballot_sync(0xFFFFFFFFu, (x >> 32) & 2u);
        const int stop = isp ? __ffs(isp) - 1 : 32;  // nearest predecessor with a prefix
        uint32_t val = lane <= stop ? (uint32_t)x : 0u;
        for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, o);
        prefix += val;
        if (isp) break;
      }
      if (lane == 0) st[tile] = (2ull << 32) | (uint32_t)(prefix + total);
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t run = s_prefix + wsum[warp] + incl - s;
  if (vec) {
    uint4* dst = reinterpret_cast<uint4*>(out + base);
#pragma unroll
    for (int q = 0; q < SCAN1_ITEMS / 4; ++q) {
      uint4 y;
      y.x = run; run += v[4 * q];
      y.y = run; run += v[4 * q + 1];
      y.z = run; run += v[4 * q + 2];
      y.w = run; run += v[4 * q + 3];
      dst[q] = y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < SCAN1_ITEMS; ++q) {
      if (base + q < len) out[base + q] = run;
      run += v[q];
    }
  }
}

}  // namespace vmps
