// engine.cuh -- leaf engine and level merge engine.
//
// Buffers: node v of the merge tree writes its output to buffer
// depth(v) mod 2 (0 = the caller's array, 1 = scratch) and reads both
// children from the other buffer, so every merge is out of place and no copy
// is ever needed (the GPU form of Pingpong's stack buffer).
//
// Leaf engine: a "unit" is a maximal subtree whose segment has <= Z elements
// (or a leaf run <= Z whose parent is larger).  Its output is the stable sort
// of its segment (a stable sort's output is unique, F1), computed
// in shared memory by a block merge sort whose merges never cross units.
// Runs longer than Z ("long leaves") are reversed (strictly descending) and/or
// copied into their parity buffer.
//
// Level engine: all non-fused nodes of one power p, as one partition launch
// (merge-path co-rank per output tile, ties from the left run, Alg. 2)
// and one merge launch (tiles staged in shared memory).
#pragma once
#include "vmps_internal.cuh"

namespace vmps {

constexpr int LEAF_THREADS = 256;
constexpr int LEAF_K = 16;
constexpr int LEAF_EMAX = 2 * MAX_FUSE_Z;  // a batch holds < 2Z elements
static_assert(LEAF_THREADS * LEAF_K == LEAF_EMAX, "leaf tile");

template <int KT>
__device__ __forceinline__ uint32_t corank(const typename KeyTraits<KT>::K* A, uint32_t nA,
                                           const typename KeyTraits<KT>::K* B, uint32_t nB,
                                           uint32_t d) {
  using T = KeyTraits<KT>;
  uint32_t lo = d > nB ? d - nB : 0u, hi = min(d, nA);
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (T::ord(A[mid]) <= T::ord(B[d - mid - 1])) lo = mid + 1;  // A[mid] precedes B[d-mid-1]
    else hi = mid;
  }
  return lo;
}

template <int KT, bool HV>
__global__ void __launch_bounds__(LEAF_THREADS) k_leaf_sort(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const uint32_t* __restrict__ units, const uint32_t* scalars, uint32_t fuse_z) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* sk = reinterpret_cast<K*>(smem_raw);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + LEAF_EMAX);
  uint16_t* us = reinterpret_cast<uint16_t*>(sv + (HV ? LEAF_EMAX : 0));
  uint16_t* ue = us + LEAF_EMAX;
  uint8_t* up = reinterpret_cast<uint8_t*>(ue + LEAF_EMAX);

  const uint32_t nunits = scalars[SC_UNITS];
  const uint32_t lo_pos = blockIdx.x * fuse_z, hi_pos = lo_pos + fuse_z;
  // units with start in [lo_pos, hi_pos)
  uint32_t x0, x1;
  {
    uint32_t a = 0, b = nunits;
    while (a < b) { uint32_t m = (a + b) >> 1; if (units[3 * m] < lo_pos) a = m + 1; else b = m; }
    x0 = a;
    b = nunits;
    while (a < b) { uint32_t m = (a + b) >> 1; if (units[3 * m] < hi_pos) a = m + 1; else b = m; }
    x1 = a;
  }
  if (x0 >= x1) return;
  const uint32_t bstart = units[3 * x0];
  const uint32_t E = units[3 * (x1 - 1) + 1] - bstart;
  for (uint32_t q = threadIdx.x; q < E; q += LEAF_THREADS) {
    sk[q] = k0[bstart + q];
    if (HV) sv[q] = v0[bstart + q];
    // unit of position q: last unit in [x0, x1) with start <= bstart + q
    uint32_t a = x0, b = x1;
    while (b - a > 1) { uint32_t m = (a + b) >> 1; if (units[3 * m] <= bstart + q) a = m; else b = m; }
    us[q] = (uint16_t)(units[3 * a] - bstart);
    ue[q] = (uint16_t)(units[3 * a + 1] - bstart);
    up[q] = (uint8_t)units[3 * a + 2];
  }
  __syncthreads();

  // Phase 1: stable odd-even transposition sort of LEAF_K consecutive
  // positions per thread, never swapping across a unit boundary.
  const uint32_t q0 = threadIdx.x * LEAF_K;
  {
    K rk[LEAF_K];
    uint32_t rv[LEAF_K];
    uint16_t ru[LEAF_K];
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) {
      uint32_t q = q0 + i;
      rk[i] = q < E ? sk[q] : K(0);
      rv[i] = (HV && q < E) ? sv[q] : 0u;
      ru[i] = q < E ? us[q] : (uint16_t)0xFFFF;
    }
#pragma unroll
    for (int rnd = 0; rnd < LEAF_K; ++rnd) {
#pragma unroll
      for (int i = rnd & 1; i + 1 < LEAF_K; i += 2) {
        bool sw = ru[i] == ru[i + 1] && T::ord(rk[i + 1]) < T::ord(rk[i]);
        if (sw) {
          K tk = rk[i]; rk[i] = rk[i + 1]; rk[i + 1] = tk;
          uint32_t tv = rv[i]; rv[i] = rv[i + 1]; rv[i + 1] = tv;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) {
      uint32_t q = q0 + i;
      if (q < E) { sk[q] = rk[i]; if (HV) sv[q] = rv[i]; }
    }
  }
  __syncthreads();

  // Phase 2: merge rounds; in the pair [x, x+2w) only the unit straddling
  // m = x + w is merged ([max(x, start), m) with [m, min(x+2w, end))); every
  // other unit of the pair is already in its final place.
  for (uint32_t w = LEAF_K; w < E; w <<= 1) {
    K rk[LEAF_K];
    uint32_t rv[LEAF_K];
    uint32_t a0 = 0, a1 = 0;
    if (q0 < E) {
      uint32_t x = (q0 / (2 * w)) * (2 * w), m = x + w;
      if (m < E && us[m] != m) {
        uint32_t lo = max(x, (uint32_t)us[m]);
        uint32_t hi = min(min(x + 2 * w, (uint32_t)ue[m]), E);
        a0 = max(q0, lo);
        a1 = min(q0 + LEAF_K, hi);
        if (a0 < a1) {
          const K* A = sk + lo;
          const K* B = sk + m;
          uint32_t nA = m - lo, nB = hi - m, d = a0 - lo;
          uint32_t ia = corank<KT>(A, nA, B, nB, d), ib = d - ia;
#pragma unroll
          for (int s = 0; s < LEAF_K; ++s) {
            if (a0 + s < a1) {
              bool takeA = ib >= nB || (ia < nA && T::ord(A[ia]) <= T::ord(B[ib]));
              if (takeA) { rk[s] = A[ia]; if (HV) rv[s] = sv[lo + ia]; ++ia; }
              else { rk[s] = B[ib]; if (HV) rv[s] = sv[m + ib]; ++ib; }
            }
          }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < LEAF_K; ++s) {
      if (a0 + s < a1) { sk[a0 + s] = rk[s]; if (HV) sv[a0 + s] = rv[s]; }
    }
    __syncthreads();
  }

  // Phase 3: each unit to its parity buffer.
  for (uint32_t q = threadIdx.x; q < E; q += LEAF_THREADS) {
    if (up[q]) { k1[bstart + q] = sk[q]; if (HV) v1[bstart + q] = sv[q]; }
    else { k0[bstart + q] = sk[q]; if (HV) v0[bstart + q] = sv[q]; }
  }
}

template <int KT>
inline size_t leaf_smem_bytes(bool hv) {
  using K = typename KeyTraits<KT>::K;
  return LEAF_EMAX * (sizeof(K) + (hv ? 4 : 0) + 2 + 2 + 1);
}

// Long leaves (> Z): reverse strictly descending runs, place odd-depth leaves
// into buffer 1.  Work is split into LONG_CHUNK pieces.
template <int KT, bool HV>
__global__ void __launch_bounds__(256) k_long_leaves(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const uint32_t* __restrict__ longs, const uint32_t* __restrict__ long_off,
    const uint32_t* scalars, uint32_t chunk) {
  using K = typename KeyTraits<KT>::K;
  const uint32_t nlong = scalars[SC_LONG];
  const uint32_t total = long_off[nlong];
  for (uint32_t c = blockIdx.x; c < total; c += gridDim.x) {
    uint32_t a = 0, b = nlong;  // last x with long_off[x] <= c
    while (b - a > 1) { uint32_t m = (a + b) >> 1; if (long_off[m] <= c) a = m; else b = m; }
    const uint32_t s = longs[4 * a], e = longs[4 * a + 1], f = longs[4 * a + 2];
    const uint32_t len = e - s;
    const bool desc = f & 2u, odd = f & 1u;
    const uint32_t base = (c - long_off[a]) * chunk;
    if (desc && !odd) {  // in-place reversal in buffer 0
      const uint32_t half = len / 2, lim = min(base + chunk, half);
      for (uint32_t q = base + threadIdx.x; q < lim; q += blockDim.x) {
        K x = k0[s + q], y = k0[e - 1 - q];
        k0[s + q] = y; k0[e - 1 - q] = x;
        if (HV) { uint32_t vx = v0[s + q], vy = v0[e - 1 - q]; v0[s + q] = vy; v0[e - 1 - q] = vx; }
      }
    } else {
      const uint32_t lim = min(base + chunk, len);
      for (uint32_t q = base + threadIdx.x; q < lim; q += blockDim.x) {
        uint32_t src = desc ? e - 1 - q : s + q;
        k1[s + q] = k0[src];
        if (HV) v1[s + q] = v0[src];
      }
    }
  }
}

// Merge-path partition of one level: co-rank at every tile start.
template <int KT>
__global__ void __launch_bounds__(256) k_partition(
    const typename KeyTraits<KT>::K* __restrict__ k0, const typename KeyTraits<KT>::K* __restrict__ k1,
    const uint32_t* __restrict__ rs, const uint32_t* __restrict__ seg_l,
    const uint32_t* __restrict__ seg_r, const uint32_t* __restrict__ dep,
    const uint32_t* __restrict__ lnodes, const uint32_t* __restrict__ ltiles,
    const uint32_t* __restrict__ level_start, const uint32_t* __restrict__ level_tile, int p,
    uint32_t tout, uint2* __restrict__ part) {
  const uint32_t ls = level_start[p], le = level_start[p + 1];
  const uint32_t tb = level_tile[p], te = level_tile[p + 1];
  for (uint32_t tau = tb + blockIdx.x * blockDim.x + threadIdx.x; tau < te;
       tau += gridDim.x * blockDim.x) {
    uint32_t a = ls, b = le;  // last x with ltiles[x] <= tau
    while (b - a > 1) { uint32_t m = (a + b) >> 1; if (ltiles[m] <= tau) a = m; else b = m; }
    const uint32_t t = lnodes[a];
    const uint32_t i = rs[seg_l[t]], j = rs[t], k = rs[seg_r[t]];
    const auto* src = (dep[t] & 1u) ? k0 : k1;
    const uint32_t d = (tau - ltiles[a]) * tout;
    part[tau - tb] = make_uint2(a, corank<KT>(src + i, j - i, src + j, k - j, d));
  }
}

// One level of stable merges, persistent over the level's tiles.
template <int KT, bool HV>
__global__ void __launch_bounds__(MERGE_BLOCK) k_merge_level(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const uint32_t* __restrict__ rs, const uint32_t* __restrict__ seg_l,
    const uint32_t* __restrict__ seg_r, const uint32_t* __restrict__ dep,
    const uint32_t* __restrict__ lnodes, const uint32_t* __restrict__ ltiles,
    const uint32_t* __restrict__ level_tile, int p, uint32_t tout,
    const uint2* __restrict__ part) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  __shared__ K sk[DEFAULT_TOUT];
  __shared__ uint32_t sv[HV ? DEFAULT_TOUT : 1];
  const uint32_t tb = level_tile[p], count = level_tile[p + 1] - tb;
  for (uint32_t tau = blockIdx.x; tau < count; tau += gridDim.x) {
    const uint2 pa = part[tau];
    const uint32_t x = pa.x, a0 = pa.y;
    const uint32_t t = lnodes[x];
    const uint32_t i = rs[seg_l[t]], j = rs[t], k = rs[seg_r[t]];
    const uint32_t nA = j - i, size = k - i;
    const uint32_t d0 = (tau + tb - ltiles[x]) * tout;
    const uint32_t d1 = min(d0 + tout, size);
    uint32_t a1 = nA;
    if (tau + 1 < count) {
      const uint2 pn = part[tau + 1];
      if (pn.x == x) a1 = pn.y;
    }
    const uint32_t b0 = d0 - a0, b1 = d1 - a1;
    const uint32_t nAw = a1 - a0, cnt = d1 - d0;
    const bool odd = dep[t] & 1u;
    const K* srck = odd ? k0 : k1;
    const uint32_t* srcv = odd ? v0 : v1;
    K* dstk = odd ? k1 : k0;
    uint32_t* dstv = odd ? v1 : v0;
    for (uint32_t q = threadIdx.x; q < cnt; q += MERGE_BLOCK) {
      uint32_t g = q < nAw ? i + a0 + q : j + b0 + (q - nAw);
      sk[q] = srck[g];
      if (HV) sv[q] = srcv[g];
    }
    __syncthreads();
    K rk[MERGE_K];
    uint32_t rv[MERGE_K];
    const uint32_t q0 = threadIdx.x * MERGE_K;
    if (q0 < cnt) {
      const K* A = sk;
      const K* B = sk + nAw;
      const uint32_t nBw = cnt - nAw;
      uint32_t ia = corank<KT>(A, nAw, B, nBw, q0), ib = q0 - ia;
#pragma unroll
      for (int s = 0; s < (int)MERGE_K; ++s) {
        bool takeA = ib >= nBw || (ia < nAw && T::ord(A[ia]) <= T::ord(B[ib]));
        if (takeA) { rk[s] = A[ia]; if (HV) rv[s] = sv[ia]; ++ia; }
        else { rk[s] = B[ib]; if (HV) rv[s] = sv[nAw + ib]; ++ib; }
      }
    }
    __syncthreads();
    if (q0 < cnt) {
#pragma unroll
      for (int s = 0; s < (int)MERGE_K; ++s) {
        if (q0 + s < cnt) { sk[q0 + s] = rk[s]; if (HV) sv[q0 + s] = rv[s]; }
      }
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < cnt; q += MERGE_BLOCK) {
      dstk[i + d0 + q] = sk[q];
      if (HV) dstv[i + d0 + q] = sv[q];
    }
    __syncthreads();
  }
}

}  // namespace vmps
