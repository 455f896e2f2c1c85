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
#include "ptx.cuh"
#include "vmps_internal.cuh"

namespace vmps {

#ifndef VMPS_LEAF_THREADS
#define VMPS_LEAF_THREADS 384
#define VMPS_LEAF_K 11
#define VMPS_LEAF_MINB 4
#endif
constexpr int LEAF_THREADS = VMPS_LEAF_THREADS;
constexpr int LEAF_K = VMPS_LEAF_K;               // odd: conflict-free chunk stride
constexpr int LEAF_CAP = LEAF_THREADS * LEAF_K;   // 4224 >= 2Z - 1 (a batch holds < 2Z)
static_assert(LEAF_CAP >= 2 * (int)MAX_FUSE_Z - 1, "leaf capacity");
constexpr int LEAF_SMALL = LEAF_THREADS / 2;          // half-size CTA for small batches
constexpr int LEAF_SMALL_CAP = LEAF_SMALL * LEAF_K;   // 2112 >= Z: any single unit fits

// The gap a - b the regula falsi interpolates: integer keys by value; f32 by
// the float values (their order images are not linear in the value), NaN
// (no interpolation) when either is not finite.
template <int KT>
__device__ __forceinline__ double interp_gap(typename KeyTraits<KT>::K a, typename KeyTraits<KT>::K b) {
  if constexpr (KT == VMPS_KEY_F32) {
    const float fa = __uint_as_float(a), fb = __uint_as_float(b);
    return (isfinite(fa) && isfinite(fb)) ? (double)fa - (double)fb : (double)NAN;
  } else {
    return (double)a - (double)b;
  }
}

// Illinois regula falsi for a bracketed search of the first m in [lo, hi]
// with g(m) > 0 (g non-decreasing; here g(m) = A[m] - B[x-m-1] on a merge
// diagonal): once both bracket ends carry a g value the probe is the
// interpolated zero crossing, the end that stays put twice has its value
// halved, and a step that does not halve the bracket is followed by a
// bisection step.  The bracket invariant is bisection's, so the result is
// exact whatever the keys; on i.i.d. keys g is near linear and a few probes
// replace log2(hi - lo).
struct RFalsi {
  double glo, ghi;
  bool klo, khi, bis;
  int side;
  __device__ __forceinline__ void init() {
    glo = ghi = 0.0;
    klo = khi = bis = false;
    side = 0;
  }
  __device__ __forceinline__ uint32_t probe(uint32_t lo, uint32_t hi, bool* interp) const {
    *interp = false;
    if (klo && khi && !bis && ghi > glo && !isnan(glo) && !isnan(ghi)) {
      const double t = -glo / (ghi - glo);  // in [0, 1]
      const double x = (double)lo - 1.0 + t * (double)(hi - lo + 1);
      *interp = true;
      return x <= (double)lo ? lo : x >= (double)(hi - 1) ? hi - 1 : (uint32_t)x;
    }
    return (lo + hi) >> 1;
  }
  // p: g(m) <= 0 at the probe m; w0 / w1 the bracket widths before / after
  __device__ __forceinline__ void update(bool p, double g, uint32_t w0, uint32_t w1, bool interp) {
    if (p) {
      glo = g; klo = true;
      if (side == 1) ghi *= 0.5;
      side = 1;
    } else {
      ghi = g; khi = true;
      if (side == 2) glo *= 0.5;
      side = 2;
    }
    bis = interp && 2 * w1 > w0;
  }
};

template <int KT>
__device__ __forceinline__ uint32_t corank(const typename KeyTraits<KT>::K* A, uint32_t nA,
                                           const typename KeyTraits<KT>::K* B, uint32_t nB,
                                           uint32_t d) {
  using T = KeyTraits<KT>;
  uint32_t lo = d > nB ? d - nB : 0u, hi = min(d, nA);
  // B[d - mid - 1] = Bd[-mid]: both probe addresses are one multiply-add
  // from mid (fewer instructions in this latency-bound loop)
  const typename KeyTraits<KT>::K* Bd = B + d - 1;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (T::ord(A[mid]) <= T::ord(Bd[-(int32_t)mid])) lo = mid + 1;  // A[mid] precedes B[d-mid-1]
    else hi = mid;
  }
  return lo;
}

// LEAF_K is odd, so thread-contiguous chunks (stride LEAF_K words) hit
// distinct banks without padding.  Shared memory carries keys and 16-bit
// local indices (ping-pong); payloads are gathered once at the end.  Rounds
// whose pairs fit inside one warp's range synchronise with __syncwarp only.
template <int KT, bool HV, int LT>
__device__ __forceinline__ void leaf_sort_batch(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const uint32_t* __restrict__ units, const uint32_t* __restrict__ batch_first, uint32_t b) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  constexpr int NTH = LT, CAP = LT * LEAF_K;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* const skb = reinterpret_cast<K*>(smem_raw);                          // 2 x CAP keys
  uint16_t* const sib = reinterpret_cast<uint16_t*>(skb + 2 * CAP);  // 2 x CAP indices
  uint32_t* ubits = reinterpret_cast<uint32_t*>(sib + 2 * CAP);      // unit-start bitmap
  uint32_t* upre = ubits + CAP / 32 + 1;  // exclusive popcount prefix per word
  uint32_t* pcar = upre + CAP / 32 + 1;   // parity of the unit open at each word's end
  uint32_t* pbits = pcar + CAP / 32 + 1;  // parity bit at each unit start

  // units of batch b (contiguous, < Zb + Z <= CAP elements)
  const uint32_t x0 = batch_first[b], x1 = batch_first[b + 1];
  if (x0 >= x1) return;
  const uint32_t bstart = units[3 * x0];
  const uint32_t E = units[3 * (x1 - 1) + 1] - bstart;
  // size classes: a batch that fits the half-size CTA goes to it (few idle
  // warps); a third, quarter-size class measured slower (one more launch)
  if (E > (uint32_t)CAP || (LT == LEAF_THREADS && E <= (uint32_t)LEAF_SMALL_CAP)) return;
  const uint32_t nwords = (E + 31) / 32;
  for (uint32_t w = threadIdx.x; w < nwords; w += NTH) { ubits[w] = 0u; pbits[w] = 0u; }
  __syncthreads();
  for (uint32_t x = x0 + threadIdx.x; x < x1; x += NTH) {
    const uint32_t q = units[3 * x] - bstart;
    atomicOr(&ubits[q >> 5], 1u << (q & 31u));
    if (units[3 * x + 2]) atomicOr(&pbits[q >> 5], 1u << (q & 31u));
  }
  const uint32_t q0 = threadIdx.x * LEAF_K;
  K rk[LEAF_K];
#pragma unroll
  for (int i = 0; i < LEAF_K; ++i) {
    const uint32_t q = q0 + i;
    rk[i] = q < E ? k0[bstart + q] : K(0);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // per-word prefix of unit starts; parity carried across words
    uint32_t carry = 0, pc = 0;
    for (uint32_t w0 = 0; w0 < nwords; w0 += 32) {
      const uint32_t w = w0 + threadIdx.x;
      const uint32_t ub = w < nwords ? ubits[w] : 0u;
      const uint32_t c = (uint32_t)__popc(ub);
      uint32_t incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)threadIdx.x >= o) incl += y;
      }
      if (w < nwords) upre[w] = carry + incl - c;
      carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
      const int hb = ub ? 31 - __clz(ub) : -1;
      const int own = hb >= 0 ? (int)((w < nwords ? pbits[w] : 0u) >> hb) & 1 : -1;
      const uint32_t has = __ballot_sync(0xFFFFFFFFu, own >= 0);
      const uint32_t le = has & (0xFFFFFFFFu >> (31 - threadIdx.x));
      const int src = le ? 31 - __clz(le) : -1;
      const int ownv = __shfl_sync(0xFFFFFFFFu, own, src >= 0 ? src : 0);
      const uint32_t pw = src >= 0 ? (uint32_t)ownv : pc;
      if (w < nwords) pcar[w] = pw;
      pc = __shfl_sync(0xFFFFFFFFu, pw, 31);
    }
  }
  __syncthreads();
  auto is_start = [&](uint32_t q) -> bool { return (ubits[q >> 5] >> (q & 31u)) & 1u; };
  auto unit_of = [&](uint32_t q) -> uint32_t {
    const uint32_t w = q >> 5;
    return upre[w] + (uint32_t)__popc(ubits[w] & (0xFFFFFFFFu >> (31u - (q & 31u)))) - 1u;
  };

  // Phase 1: stable rank sort of the thread's chunk by (unit, key).
  {
    uint32_t cut[LEAF_K];
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) {
      const uint32_t q = q0 + i;
      if (i > 0 && q < E && is_start(q)) ++c;
      cut[i] = q < E ? c : 0xFFu;  // past-E elements rank last
    }
    uint32_t rank[LEAF_K];
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) rank[i] = 0;
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) {
#pragma unroll
      for (int j = i + 1; j < LEAF_K; ++j) {
        const bool ifirst = cut[i] != cut[j] || T::ord(rk[i]) <= T::ord(rk[j]);
        rank[j] += ifirst ? 1u : 0u;
        rank[i] += ifirst ? 0u : 1u;
      }
    }
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) {
      if (q0 + i < E) {
        skb[q0 + rank[i]] = rk[i];
        sib[q0 + rank[i]] = (uint16_t)(q0 + i);
      }
    }
  }
  __syncthreads();

  // Phase 2: merge rounds (ping-pong).  In the pair [x, x+2w) only the unit
  // straddling m = x + w is merged ([max(x, start), m) with
  // [m, min(x+2w, end))); everything else is copied in place.
  uint32_t cur = 0;
  for (uint32_t w = LEAF_K; w < E; w <<= 1) {
    const K* sk = skb + cur * CAP;
    const uint16_t* si = sib + cur * CAP;
    K* dk = skb + (cur ^ 1u) * CAP;
    uint16_t* di = sib + (cur ^ 1u) * CAP;
    if (q0 < E) {
      const uint32_t q1 = min(q0 + LEAF_K, E);
      const uint32_t x = (q0 / (2 * w)) * (2 * w), m = x + w;
      uint32_t a0 = q0, a1 = q0, lo = 0, hi = 0;
      if (m < E && !is_start(m)) {
        const uint32_t* u = units + 3 * (x0 + unit_of(m));
        lo = max(x, u[0] - bstart);
        hi = min(min(x + 2 * w, u[1] - bstart), E);
        a0 = max(q0, lo);
        a1 = max(a0, min(q1, hi));
      }
      uint32_t ri[LEAF_K];
      if (a0 == q0 && a1 == q0 + LEAF_K) {
        // the whole chunk lies in the merge window: branch-free serial merge
        const uint32_t nA = m - lo, nB = hi - m, d = q0 - lo;
        uint32_t l = d > nB ? d - nB : 0u, h = min(d, nA);
        while (l < h) {
          const uint32_t mid = (l + h) >> 1;
          if (T::ord(sk[lo + mid]) <= T::ord(sk[m + d - mid - 1])) l = mid + 1;
          else h = mid;
        }
        uint32_t ia = lo + l, ib = m + d - l;  // absolute positions
        // heads and one-ahead prefetches of both sides (reads past a side stay
        // inside the buffer and are never used)
        K ka = sk[ia], kb = sk[ib], ka2 = sk[ia + 1], kb2 = sk[ib + 1];
#pragma unroll
        for (int s2 = 0; s2 < LEAF_K; ++s2) {
          const bool p = ib >= hi || (ia < m && T::ord(ka) <= T::ord(kb));
          rk[s2] = p ? ka : kb;
          ri[s2] = p ? ia : ib;
          ia += p ? 1u : 0u;
          ib += p ? 0u : 1u;
          const K nx = sk[(p ? ia : ib) + 1];
          ka = p ? ka2 : ka;
          kb = p ? kb : kb2;
          ka2 = p ? nx : ka2;
          kb2 = p ? kb2 : nx;
        }
#pragma unroll
        for (int s2 = 0; s2 < LEAF_K; ++s2) {
          dk[q0 + s2] = rk[s2];
          di[q0 + s2] = si[ri[s2]];
        }
      } else if (a0 >= a1) {  // nothing to merge here: copy in place
#pragma unroll
        for (int s2 = 0; s2 < LEAF_K; ++s2) {
          const uint32_t pos = q0 + s2;
          if (pos < q1) { dk[pos] = sk[pos]; di[pos] = si[pos]; }
        }
      } else {  // the chunk holds a unit boundary: mixed merge / copy
        const uint32_t nA = m - lo, nB = hi - m, d = a0 - lo;
        uint32_t l = d > nB ? d - nB : 0u, h = min(d, nA);
        while (l < h) {
          const uint32_t mid = (l + h) >> 1;
          if (T::ord(sk[lo + mid]) <= T::ord(sk[m + d - mid - 1])) l = mid + 1;
          else h = mid;
        }
        uint32_t ia = l, ib = d - l;
        K ka = sk[lo + min(ia, nA - 1)];
        K kb = sk[m + min(ib, nB - 1)];
#pragma unroll
        for (int s2 = 0; s2 < LEAF_K; ++s2) {
          const uint32_t pos = q0 + s2;
          if (pos >= a0 && pos < a1) {
            const bool takeA = ib >= nB || (ia < nA && T::ord(ka) <= T::ord(kb));
            if (takeA) {
              rk[s2] = ka; ri[s2] = lo + ia; ++ia;
              if (ia < nA) ka = sk[lo + ia];
            } else {
              rk[s2] = kb; ri[s2] = m + ib; ++ib;
              if (ib < nB) kb = sk[m + ib];
            }
          } else {
            rk[s2] = pos < q1 ? sk[pos] : K(0);
            ri[s2] = pos;
          }
        }
#pragma unroll
        for (int s2 = 0; s2 < LEAF_K; ++s2) {
          const uint32_t pos = q0 + s2;
          if (pos < q1) { dk[pos] = rk[s2]; di[pos] = si[ri[s2]]; }
        }
      }
    }
    cur ^= 1u;
    // the next round's pairs stay inside one warp's range: warp-level sync
    if (2 * (2 * w) <= 32 * LEAF_K) __syncwarp();
    else __syncthreads();
  }
  __syncthreads();

  // Phase 3: keys from shared memory, payloads gathered by local index (read
  // all before writing: the payload gather may be in place), each unit to its
  // parity buffer.
  const K* sk = skb + cur * CAP;
  const uint16_t* si = sib + cur * CAP;
  constexpr int PER = CAP / NTH;
  uint32_t gv[PER];
  if (HV) {
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t q = threadIdx.x + r * NTH;
      gv[r] = q < E ? v0[bstart + si[q]] : 0u;
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const uint32_t q = threadIdx.x + r * NTH;
    if (q < E) {
      const uint32_t w = q >> 5;
      const uint32_t mk = ubits[w] & (0xFFFFFFFFu >> (31u - (q & 31u)));
      const uint32_t par = mk ? (pbits[w] >> (31 - __clz(mk))) & 1u : pcar[w - 1];
      if (par) { k1[bstart + q] = sk[q]; if (HV) v1[bstart + q] = gv[r]; }
      else { k0[bstart + q] = sk[q]; if (HV) v0[bstart + q] = gv[r]; }
    }
  }
}

// ---------------------------------------------------------------------------
// Composite-key leaf (4-byte keys, VMPS_LEAF_C): every element of the batch
// becomes one u64 c = unit ordinal (19 bits) | order image of the key (32) |
// batch position (13).  The units of a batch are consecutive and a unit's
// fused subtree ends as the stable sort of its elements (Alg. 1's merges of
// sorted runs, ties to the left run, keep equal keys in input order),
// so the whole batch sorted by c is exactly every unit's result in place --
// and the c are distinct, so the rounds below are plain merges of one u64
// stream: no unit boundaries inside the rounds (no unit lookups, no mixed
// merge / copy chunks), no separate index array to gather each round, and
// the payload is gathered once at the end by the position bits.  Positions
// [E, Ep) hold all-ones sentinels (Ep = E rounded up to LEAF_K).
// ---------------------------------------------------------------------------
#ifndef VMPS_LEAF_C
#define VMPS_LEAF_C 1
#endif
#ifndef VMPS_LEAF_SKIP
#define VMPS_LEAF_SKIP 1
#endif
template <int KT>
__host__ __device__ constexpr bool leaf_composite() {
  return VMPS_LEAF_C && sizeof(typename KeyTraits<KT>::K) == 4;
}
// resident CTAs of the full-size class per SM (the half-size class: twice as many)
template <int KT>
__host__ __device__ constexpr int leaf_minb() { return leaf_composite<KT>() ? 3 : VMPS_LEAF_MINB; }

template <int KT, bool HV, int LT>
__device__ __forceinline__ void leaf_sort_batch_c(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const uint32_t* __restrict__ units, const uint32_t* __restrict__ batch_first, uint32_t b) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  static_assert(sizeof(K) == 4, "composite leaf: 4-byte keys");
  static_assert(LT * LEAF_K <= 8192, "composite leaf: 13 position bits");
  constexpr int NTH = LT, CAP = LT * LEAF_K;
  constexpr uint64_t SENT = ~0ull;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* const scb = reinterpret_cast<uint64_t*>(smem_raw);  // 2 x CAP composites
  uint32_t* ubits = reinterpret_cast<uint32_t*>(scb + 2 * CAP);  // unit-start bitmap
  uint32_t* upre = ubits + CAP / 32 + 1;  // exclusive popcount prefix per word
  uint32_t* pcar = upre + CAP / 32 + 1;   // parity of the unit open at each word's end
  uint32_t* pbits = pcar + CAP / 32 + 1;  // parity bit at each unit start

  const uint32_t x0 = batch_first[b], x1 = batch_first[b + 1];
  if (x0 >= x1) return;
  const uint32_t bstart = units[3 * x0];
  const uint32_t E = units[3 * (x1 - 1) + 1] - bstart;
  if (E > (uint32_t)CAP || (LT == LEAF_THREADS && E <= (uint32_t)LEAF_SMALL_CAP)) return;
  const uint32_t nwords = (E + 31) / 32;
  for (uint32_t w = threadIdx.x; w < nwords; w += NTH) { ubits[w] = 0u; pbits[w] = 0u; }
  __syncthreads();
  for (uint32_t x = x0 + threadIdx.x; x < x1; x += NTH) {
    const uint32_t q = units[3 * x] - bstart;
    atomicOr(&ubits[q >> 5], 1u << (q & 31u));
    if (units[3 * x + 2]) atomicOr(&pbits[q >> 5], 1u << (q & 31u));
  }
  const uint32_t q0 = threadIdx.x * LEAF_K;
  K rk[LEAF_K];
#pragma unroll
  for (int i = 0; i < LEAF_K; ++i) {
    const uint32_t q = q0 + i;
    rk[i] = q < E ? k0[bstart + q] : K(0);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // per-word prefix of unit starts; parity carried across words
    uint32_t carry = 0, pc = 0;
    for (uint32_t w0 = 0; w0 < nwords; w0 += 32) {
      const uint32_t w = w0 + threadIdx.x;
      const uint32_t ub = w < nwords ? ubits[w] : 0u;
      const uint32_t c = (uint32_t)__popc(ub);
      uint32_t incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)threadIdx.x >= o) incl += y;
      }
      if (w < nwords) upre[w] = carry + incl - c;
      carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
      const int hb = ub ? 31 - __clz(ub) : -1;
      const int own = hb >= 0 ? (int)((w < nwords ? pbits[w] : 0u) >> hb) & 1 : -1;
      const uint32_t has = __ballot_sync(0xFFFFFFFFu, own >= 0);
      const uint32_t le = has & (0xFFFFFFFFu >> (31 - threadIdx.x));
      const int src = le ? 31 - __clz(le) : -1;
      const int ownv = __shfl_sync(0xFFFFFFFFu, own, src >= 0 ? src : 0);
      const uint32_t pw = src >= 0 ? (uint32_t)ownv : pc;
      if (w < nwords) pcar[w] = pw;
      pc = __shfl_sync(0xFFFFFFFFu, pw, 31);
    }
  }
  __syncthreads();

  // Phase 1: composites of the thread's chunk, stable rank sort, into buffer 0.
  const uint32_t Ep = (E + LEAF_K - 1) / LEAF_K * LEAF_K;
  if (q0 < E) {
    uint32_t u;
    {
      const uint32_t w = q0 >> 5;
      u = upre[w] + (uint32_t)__popc(ubits[w] & (0xFFFFFFFFu >> (31u - (q0 & 31u)))) - 1u;
    }
    uint64_t c[LEAF_K];
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) {
      const uint32_t q = q0 + i;
      if (i > 0 && q < E && ((ubits[q >> 5] >> (q & 31u)) & 1u)) ++u;
      c[i] = q < E ? ((uint64_t)u << 45) | ((uint64_t)T::ord(rk[i]) << 13) | (uint64_t)q : SENT;
    }
    uint32_t rank[LEAF_K];
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) rank[i] = 0;
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) {
#pragma unroll
      for (int j = i + 1; j < LEAF_K; ++j) {
        const bool ifirst = c[i] <= c[j];
        rank[j] += ifirst ? 1u : 0u;
        rank[i] += ifirst ? 0u : 1u;
      }
    }
#pragma unroll
    for (int i = 0; i < LEAF_K; ++i) scb[q0 + rank[i]] = c[i];
  }
  __syncthreads();

  // Phase 2: merge rounds over [0, Ep) (ping-pong): pairs [x, x+w) + [x+w, x+2w).
  uint32_t cur = 0;
  for (uint32_t w = LEAF_K, wc = 1; w < E; w <<= 1, wc <<= 1) {  // wc = w / LEAF_K chunks
    const uint64_t* sk = scb + cur * CAP;
    uint64_t* dk = scb + (cur ^ 1u) * CAP;
    if (q0 < Ep) {
      const uint32_t x = (threadIdx.x & ~(2 * wc - 1)) * LEAF_K, m = x + w;  // pair start, no division
      // a pair already in order (A's last <= B's first: presorted stretches)
      // is its own merge: copy, no search
      if (m < Ep && !(VMPS_LEAF_SKIP && sk[m - 1] <= sk[m])) {
        const uint32_t hi = min(x + 2 * w, Ep), nB = hi - m, d = q0 - x;
        uint32_t l = d > nB ? d - nB : 0u, h = min(d, w);
        while (l < h) {
          const uint32_t mid = (l + h) >> 1;
          if (sk[x + mid] <= sk[m + d - mid - 1]) l = mid + 1;
          else h = mid;
        }
        uint32_t ia = x + l, ib = m + d - l;  // absolute positions
        uint64_t ka = sk[ia], kb = sk[ib];     // a read at hi stays inside shared memory, unused
        uint64_t o[LEAF_K];
#pragma unroll
        for (int s2 = 0; s2 < LEAF_K; ++s2) {
          const bool p = ib >= hi || (ia < m && ka <= kb);
          o[s2] = p ? ka : kb;
          ia += p ? 1u : 0u;
          ib += p ? 0u : 1u;
          const uint64_t nx = sk[p ? ia : ib];
          ka = p ? nx : ka;
          kb = p ? kb : nx;
        }
#pragma unroll
        for (int s2 = 0; s2 < LEAF_K; ++s2) dk[q0 + s2] = o[s2];
      } else {  // no partner, or the pair is in order: copy
#pragma unroll
        for (int s2 = 0; s2 < LEAF_K; ++s2) dk[q0 + s2] = sk[q0 + s2];
      }
    }
    cur ^= 1u;
    // the next round's pairs stay inside one warp's range: warp-level sync
    if (2 * (2 * w) <= 32 * LEAF_K) __syncwarp();
    else __syncthreads();
  }
  __syncthreads();

  // Phase 3: keys (u32: from the composite; f32: gathered, the order image of
  // NaNs is not invertible) and payloads gathered by position, each unit to
  // its parity buffer.  The batch's payloads (and f32 keys) are first read
  // coalesced into the free ping-pong buffer -- all global reads precede the
  // barrier, so the in-place writes below cannot overtake them -- and
  // gathered from shared memory.
  const uint64_t* sk = scb + cur * CAP;
  constexpr int PER = CAP / NTH;
  constexpr bool GK = KT != VMPS_KEY_U32;
  uint32_t* sv = reinterpret_cast<uint32_t*>(scb + (cur ^ 1u) * CAP);  // 2 CAP words: values, then f32 keys
  if (HV || GK) {
    for (uint32_t q = threadIdx.x; q < E; q += NTH) {
      if (HV) sv[q] = v0[bstart + q];
      if (GK) sv[CAP + q] = (uint32_t)k0[bstart + q];
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const uint32_t q = threadIdx.x + r * NTH;
    if (q < E) {
      const uint64_t c = sk[q];
      const uint32_t src = (uint32_t)c & 0x1FFFu;
      const K gk = GK ? (K)sv[CAP + src] : (K)(uint32_t)(c >> 13);
      const uint32_t gv = HV ? sv[src] : 0u;
      const uint32_t w = q >> 5;
      const uint32_t mk = ubits[w] & (0xFFFFFFFFu >> (31u - (q & 31u)));
      const uint32_t par = mk ? (pbits[w] >> (31 - __clz(mk))) & 1u : pcar[w - 1];
      if (par) { k1[bstart + q] = gk; if (HV) v1[bstart + q] = gv; }
      else { k0[bstart + q] = gk; if (HV) v0[bstart + q] = gv; }
    }
  }
}

// Persistent CTAs take batches from a work queue (atomic counter per size
// class), so every resident CTA stays busy and no CTA is launched per empty
// slot of the batch bound.
template <int KT, bool HV, int LT>
__global__ void __launch_bounds__(LT, leaf_minb<KT>() * (LEAF_THREADS / LT)) k_leaf_sort(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const uint32_t* __restrict__ units, const uint32_t* __restrict__ batch_first, uint32_t* scalars) {
  __shared__ uint32_t s_b;
  const uint32_t nb = scalars[SC_NBATCH];
  uint32_t* q = scalars + (LT == LEAF_THREADS ? SC_LEAFQ1 : SC_LEAFQ);
  for (;;) {
    if (threadIdx.x == 0) s_b = atomicAdd(q, 1u);
    __syncthreads();
    const uint32_t b = s_b;
    if (b >= nb) break;
    if constexpr (leaf_composite<KT>()) leaf_sort_batch_c<KT, HV, LT>(k0, v0, k1, v1, units, batch_first, b);
    else leaf_sort_batch<KT, HV, LT>(k0, v0, k1, v1, units, batch_first, b);
    __syncthreads();  // shared memory (and s_b) are reused by the next batch
  }
}

template <int KT, int LT = LEAF_THREADS>
inline size_t leaf_smem_bytes(bool hv) {
  using K = typename KeyTraits<KT>::K;
  (void)hv;
  constexpr int CAP = LT * LEAF_K;
  if (leaf_composite<KT>()) return 2 * CAP * 8 + 4 * (CAP / 32 + 1) * 4 + 16;
  return 2 * CAP * (sizeof(K) + 2) + 4 * (CAP / 32 + 1) * 4 + 16;
}

// Leaf batches: consecutive units that start in the same window of Zb
// positions and touch (no long leaf between them).  flag[x] = unit x opens a
// batch; zero tail up to cap so the scan sees a clean array.
__global__ void k_batch_flags(const uint32_t* __restrict__ units, const uint32_t* scalars, uint32_t zb,
                              uint32_t cap, uint32_t* __restrict__ flag) {
  const uint32_t nunits = scalars[SC_UNITS];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= cap; x += gridDim.x * blockDim.x) {
    uint32_t f = 0;
    if (x < nunits) {
      const uint32_t s = units[3 * x];
      f = x == 0 || s / zb != units[3 * (x - 1)] / zb || s != units[3 * (x - 1) + 1];
    }
    flag[x] = f;
  }
}

// batch_first[b] = first unit of batch b; batch_first[b] = nunits for every
// b >= the batch count up to bcap (those CTAs exit at once).
__global__ void k_batch_first(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ idx,
                              uint32_t* scalars, uint32_t bcap, uint32_t* __restrict__ batch_first) {
  const uint32_t nunits = scalars[SC_UNITS];
  const uint32_t nb = idx[nunits];
  if (blockIdx.x == 0 && threadIdx.x == 0) scalars[SC_NBATCH] = nb;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < nunits; x += gridDim.x * blockDim.x)
    if (flag[x]) batch_first[idx[x]] = x;
  for (uint32_t b = nb + blockIdx.x * blockDim.x + threadIdx.x; b <= bcap; b += gridDim.x * blockDim.x)
    batch_first[b] = nunits;
}

#ifndef VMPS_LONG_U
#define VMPS_LONG_U 8  // elements per thread in flight per batch of a long-leaf copy
#endif
#ifndef VMPS_LONG_MINB
#define VMPS_LONG_MINB 4  // resident CTAs per SM (caps registers at 64: 80 left 3 CTAs; 6 and 8 spill)
#endif
// Long leaves (> Z): reverse strictly descending runs, place odd-depth leaves
// into buffer 1.  Work is split into LONG_CHUNK pieces.
template <int KT, bool HV>
__global__ void __launch_bounds__(256, VMPS_LONG_MINB) k_long_leaves(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const uint32_t* __restrict__ longs, const uint32_t* __restrict__ long_off,
    const uint32_t* scalars, uint32_t chunk) {
  using K = typename KeyTraits<KT>::K;
  const uint32_t nlong = scalars[SC_LONG];
  const uint32_t total = long_off[nlong];
  // a contiguous range of chunks per CTA: one search for the first chunk's
  // leaf, then the leaf index only moves forward (a search per chunk was a
  // chain of ~17 dependent loads per 4096 elements)
  const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint32_t c0 = blockIdx.x * per, c1 = min(total, c0 + per);
  uint32_t a = 0;
  if (c0 < c1) {
    uint32_t b = nlong;  // last x with long_off[x] <= c0
    while (b - a > 1) { uint32_t m = (a + b) >> 1; if (long_off[m] <= c0) a = m; else b = m; }
  }
  for (uint32_t c = c0; c < c1; ++c) {
    while (a + 1 < nlong && long_off[a + 1] <= c) ++a;
    const uint32_t s = longs[4 * a], e = longs[4 * a + 1], f = longs[4 * a + 2];
    const uint32_t len = e - s;
    const bool desc = f & 2u, odd = f & 1u;
    const uint32_t base = (c - long_off[a]) * chunk;
    // U independent elements per thread in flight (loads first, then stores);
    // the reversal holds two of each (both ends), so half as many
    constexpr int U = VMPS_LONG_U;
    if (desc && !odd) {  // in-place reversal in buffer 0
      constexpr int UR = U / 2;
      const uint32_t half = len / 2, lim = min(base + chunk, half);
      for (uint32_t q0 = base + threadIdx.x; q0 < lim; q0 += UR * blockDim.x) {
        K x[UR], y[UR];
        uint32_t vx[UR], vy[UR];
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const uint32_t q = q0 + u * blockDim.x;
          if (q < lim) {
            x[u] = k0[s + q]; y[u] = k0[e - 1 - q];
            if (HV) { vx[u] = v0[s + q]; vy[u] = v0[e - 1 - q]; }
          }
        }
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const uint32_t q = q0 + u * blockDim.x;
          if (q < lim) {
            k0[s + q] = y[u]; k0[e - 1 - q] = x[u];
            if (HV) { v0[s + q] = vy[u]; v0[e - 1 - q] = vx[u]; }
          }
        }
      }
    } else {
      const uint32_t lim = min(base + chunk, len);
      for (uint32_t q0 = base + threadIdx.x; q0 < lim; q0 += U * blockDim.x) {
        K x[U];
        uint32_t vx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t q = q0 + u * blockDim.x;
          if (q < lim) {
            const uint32_t src = desc ? e - 1 - q : s + q;
            x[u] = k0[src];
            if (HV) vx[u] = v0[src];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t q = q0 + u * blockDim.x;
          if (q < lim) { k1[s + q] = x[u]; if (HV) v1[s + q] = vx[u]; }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Level engine.  Output tiles are aligned to global positions: tile g of a
// node [i,k) covers [max(i, g T), min(k, (g+1) T)), so every interior tile
// starts on a T-element boundary and threads store 128-bit vectors.
// ---------------------------------------------------------------------------
struct __align__(16) TileDesc {
  uint32_t i, j, k;  // the node's merge [i,j) + [j,k)
  uint32_t lo, hi;   // output range of this tile
  uint32_t a0, a1;   // elements of [i,j) among outputs [i,lo) / [i,hi)
  uint32_t par;      // output buffer (depth parity)
};

// Warp-cooperative merge-path co-rank (32-ary search, ties to A): the number
// of A elements among the first d outputs of merging A[0,nA) and B[0,nB).
template <int KT>
__device__ __forceinline__ uint32_t warp_corank(const typename KeyTraits<KT>::K* A, uint32_t nA,
                                                const typename KeyTraits<KT>::K* B, uint32_t nB,
                                                uint32_t d, int lane) {
  using T = KeyTraits<KT>;
  uint32_t lo = d > nB ? d - nB : 0u, hi = min(d, nA);
  // invariant: answer in [lo, hi]; P(m) = A[m] <= B[d-m-1] is true below it
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t m = lo + (uint32_t)lane * step + step - 1;
    const bool valid = m < hi;
    const bool pr = valid && T::ord(A[m]) <= T::ord(B[d - m - 1]);
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, pr);
    const uint32_t vb = __ballot_sync(0xFFFFFFFFu, valid);
    const int c = __popc(bal);
    const uint32_t mc1 = __shfl_sync(0xFFFFFFFFu, m, c > 0 ? c - 1 : 0);
    const uint32_t mc = __shfl_sync(0xFFFFFFFFu, m, c < 32 ? c : 31);
    const int nv = __popc(vb);
    const uint32_t nlo = c > 0 ? mc1 + 1 : lo;
    const uint32_t nhi = c < nv ? mc : hi;
    lo = nlo;
    hi = nhi;
  }
  const uint32_t m = lo + (uint32_t)lane;
  const bool pr = m < hi && T::ord(A[m]) <= T::ord(B[d - m - 1]);
  return lo + (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, pr));
}

// Bounded merge-path co-rank: the answer is known to lie in [lb, ub].
template <int KT>
__device__ __forceinline__ uint32_t corank_in(const typename KeyTraits<KT>::K* A, uint32_t nA,
                                              const typename KeyTraits<KT>::K* B, uint32_t nB,
                                              uint32_t d, uint32_t lb, uint32_t ub) {
  using T = KeyTraits<KT>;
  uint32_t lo = max(d > nB ? d - nB : 0u, lb), hi = min(min(d, nA), ub);
  const typename KeyTraits<KT>::K* Bd = B + d - 1;  // B[d - mid - 1] = Bd[-mid]
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (T::ord(A[mid]) <= T::ord(Bd[-(int32_t)mid])) lo = mid + 1;  // A[mid] precedes B[d-mid-1]
    else hi = mid;
  }
  return lo;
}

// Tile descriptors of one level.  A thread handles DESC_CHUNK consecutive
// tiles: the first co-rank is a full binary search, each next tile of the
// same node searches only [a0, a0 + T] (co-ranks are monotone and grow by at
// most the diagonal step), so most probes stay inside a few DRAM lines.
constexpr uint32_t DESC_CHUNK = 4;
template <int KT>
__global__ void __launch_bounds__(256) k_tile_desc(
    const typename KeyTraits<KT>::K* __restrict__ k0, const typename KeyTraits<KT>::K* __restrict__ k1,
    const uint32_t* __restrict__ rs, const uint32_t* __restrict__ seg_l,
    const uint32_t* __restrict__ seg_r, const uint32_t* __restrict__ dep,
    const uint32_t* __restrict__ lnodes, const uint32_t* __restrict__ ltiles,
    const uint32_t* __restrict__ level_start, const uint32_t* __restrict__ level_tile, int p,
    uint32_t tout, TileDesc* __restrict__ desc, uint32_t cap, uint32_t* scalars) {
  const uint32_t ls = level_start[p], le = level_start[p + 1];
  const uint32_t tb = level_tile[p], te = level_tile[p + 1];
  if (te - tb > cap) {  // never expected: the bound in carve() is exact
    if (blockIdx.x == 0 && threadIdx.x == 0) scalars[SC_ERROR] = 2;
    return;
  }
  const uint32_t nchunks = (te - tb + DESC_CHUNK - 1) / DESC_CHUNK;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += gridDim.x * blockDim.x) {
    const uint32_t tau0 = tb + c * DESC_CHUNK;
    uint32_t a = ls, b = le;  // last bucket x with ltiles[x] <= tau0
    while (b - a > 1) { uint32_t m = (a + b) >> 1; if (ltiles[m] <= tau0) a = m; else b = m; }
    uint32_t cur_node = 0xFFFFFFFFu, prev_a0 = 0, prev_lo = 0;
    for (uint32_t q = 0; q < DESC_CHUNK; ++q) {
      const uint32_t tau = tau0 + q;
      if (tau >= te) break;
      while (a + 1 < le && ltiles[a + 1] <= tau) ++a;
      const uint32_t t = lnodes[a];
      const uint32_t i = rs[seg_l[t]], j = rs[t], k = rs[seg_r[t]];
      const uint32_t par = dep[t] & 1u;
      const uint32_t g = i / tout + (tau - ltiles[a]);
      const uint32_t lo = max(i, g * tout), hi = min(k, (g + 1) * tout);
      const auto* src = par ? k0 : k1;
      uint32_t lb = 0, ub = 0xFFFFFFFFu;
      if (cur_node == a) { lb = prev_a0; ub = prev_a0 + (lo - prev_lo); }
      const uint32_t a0 = corank_in<KT>(src + i, j - i, src + j, k - j, lo - i, lb, ub);
      cur_node = a; prev_a0 = a0; prev_lo = lo;
      TileDesc* D = desc + (tau - tb);
      D->i = i; D->j = j; D->k = k; D->lo = lo; D->hi = hi; D->a0 = a0; D->par = par;
      if (hi == k) D->a1 = j - i;
      if (lo != i) desc[tau - tb - 1].a1 = a0;
    }
  }
}

constexpr uint32_t MERGE_STAGES = 2;  // tiles in flight per CTA = MERGE_STAGES - 1

template <int KT, bool HV>
struct MergeSmem {
  using K = typename KeyTraits<KT>::K;
  static constexpr uint32_t KB = DEFAULT_TOUT * sizeof(K) + 64;
  static constexpr uint32_t VB = HV ? DEFAULT_TOUT * 4 + 64 : 0;
  static constexpr uint32_t STAGE = KB + VB;
  static constexpr uint32_t HDR = 256;  // mbarriers at 0, MergeHdr (48 B) per stage at 64
  static constexpr uint32_t BYTES = HDR + MERGE_STAGES * STAGE;
};

struct MergeHdr {
  uint32_t a_base, nA, b_base, nB;    // key element offsets in the stage
  uint32_t va_base, vb_base, lo, hi;  // value element offsets, output range
  uint32_t par, pad[3];
};
static_assert(64 + MERGE_STAGES * sizeof(MergeHdr) <= 256 && MERGE_STAGES * 8 <= 64, "merge smem header area");

// Thread 0: fetch tile `tau` into stage `s` with 1-D bulk copies over the
// 16-byte-aligned superset of each window (reads never cross a page).
template <int KT, bool HV>
__device__ __forceinline__ void merge_issue(const TileDesc& d, uint32_t s, unsigned char* smem, uint64_t* bars,
                                            MergeHdr* hdr, const typename KeyTraits<KT>::K* k0, const uint32_t* v0,
                                            const typename KeyTraits<KT>::K* k1, const uint32_t* v1) {
  using SM = MergeSmem<KT, HV>;
  using K = typename KeyTraits<KT>::K;
  const K* sk = d.par ? k0 : k1;
  const uint32_t* sv = d.par ? v0 : v1;
  const uint32_t nA = d.a1 - d.a0, cnt = d.hi - d.lo, nB = cnt - nA;
  const uint32_t aoff = d.i + d.a0, boff = d.j + (d.lo - d.i) - d.a0;
  unsigned char* st = smem + SM::HDR + s * SM::STAGE;
  uint32_t total = 0;
  MergeHdr h;
  // keys
  {
    const uintptr_t ga = (uintptr_t)(sk + aoff), ga0 = ga & ~(uintptr_t)15;
    const uint32_t bA = nA ? (uint32_t)(((ga + (uintptr_t)nA * sizeof(K) + 15) & ~(uintptr_t)15) - ga0) : 0u;
    const uintptr_t gb = (uintptr_t)(sk + boff), gb0 = gb & ~(uintptr_t)15;
    const uint32_t bB = nB ? (uint32_t)(((gb + (uintptr_t)nB * sizeof(K) + 15) & ~(uintptr_t)15) - gb0) : 0u;
    h.a_base = (uint32_t)(ga - ga0) / sizeof(K);
    h.b_base = (bA + (uint32_t)(gb - gb0)) / sizeof(K);
    h.nA = nA;
    h.nB = nB;
    if (bA) { total += bA; }
    if (bB) { total += bB; }
    if (HV) {
      const uintptr_t va = (uintptr_t)(sv + aoff), va0 = va & ~(uintptr_t)15;
      const uint32_t vA = nA ? (uint32_t)(((va + (uintptr_t)nA * 4 + 15) & ~(uintptr_t)15) - va0) : 0u;
      const uintptr_t vb = (uintptr_t)(sv + boff), vb0 = vb & ~(uintptr_t)15;
      const uint32_t vB = nB ? (uint32_t)(((vb + (uintptr_t)nB * 4 + 15) & ~(uintptr_t)15) - vb0) : 0u;
      h.va_base = (uint32_t)(va - va0) / 4;
      h.vb_base = (vA + (uint32_t)(vb - vb0)) / 4;
      total += vA + vB;
      h.lo = d.lo; h.hi = d.hi; h.par = d.par;
      hdr[s] = h;
      mbar_arrive_expect_tx(&bars[s], total);
      if (bA) bulk_g2s(st, (const void*)ga0, bA, &bars[s]);
      if (bB) bulk_g2s(st + bA, (const void*)gb0, bB, &bars[s]);
      if (vA) bulk_g2s(st + SM::KB, (const void*)va0, vA, &bars[s]);
      if (vB) bulk_g2s(st + SM::KB + vA, (const void*)vb0, vB, &bars[s]);
    } else {
      h.va_base = h.vb_base = 0;
      h.lo = d.lo; h.hi = d.hi; h.par = d.par;
      hdr[s] = h;
      mbar_arrive_expect_tx(&bars[s], total);
      if (bA) bulk_g2s(st, (const void*)ga0, bA, &bars[s]);
      if (bB) bulk_g2s(st + bA, (const void*)gb0, bB, &bars[s]);
    }
  }
}

template <typename K>
__device__ __forceinline__ void store_vec8(K* dst, const K (&r)[MERGE_K]);
template <>
__device__ __forceinline__ void store_vec8<uint32_t>(uint32_t* dst, const uint32_t (&r)[MERGE_K]) {
#pragma unroll
  for (int q = 0; q < (int)MERGE_K; q += 4) st_v4(dst + q, r[q], r[q + 1], r[q + 2], r[q + 3]);
}
template <>
__device__ __forceinline__ void store_vec8<uint64_t>(uint64_t* dst, const uint64_t (&r)[MERGE_K]) {
#pragma unroll
  for (int q = 0; q < (int)MERGE_K; q += 2)
    st_v4(dst + q, (uint32_t)r[q], (uint32_t)(r[q] >> 32), (uint32_t)r[q + 1], (uint32_t)(r[q + 1] >> 32));
}

// One level of stable merges: persistent CTAs, double-buffered bulk copies,
// merge-path inside the tile, 128-bit stores.
template <int KT, bool HV>
__global__ void __launch_bounds__(MERGE_BLOCK, 3) k_merge_level(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const TileDesc* __restrict__ desc, const uint32_t* __restrict__ level_tile, int p, uint32_t tout,
    uint32_t cap) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  using SM = MergeSmem<KT, HV>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  MergeHdr* hdr = reinterpret_cast<MergeHdr*>(smem + 64);
  const uint32_t count = level_tile[p + 1] - level_tile[p];
  if (blockIdx.x >= count || count > cap) return;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    for (uint32_t q = 0; q < MERGE_STAGES; ++q) mbar_init(&bars[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // thread 0 keeps the descriptor of the next tile to issue in registers, one
  // issue ahead, so a bulk copy never waits for its descriptor load
  TileDesc dn;
  if (tid == 0) {
    for (uint32_t q = 0; q + 1 < MERGE_STAGES; ++q)
      if (blockIdx.x + q * gridDim.x < count)
        merge_issue<KT, HV>(desc[blockIdx.x + q * gridDim.x], q, smem, bars, hdr, k0, v0, k1, v1);
    const uint32_t f = blockIdx.x + (MERGE_STAGES - 1) * gridDim.x;
    if (f < count) dn = desc[f];
  }
  uint32_t it = 0;
  for (uint32_t tau = blockIdx.x; tau < count; tau += gridDim.x, ++it) {
    const uint32_t s = it % MERGE_STAGES;
    // refill the stage consumed in the previous iteration (freed by its barrier)
    const uint32_t ahead = tau + (MERGE_STAGES - 1) * gridDim.x;
    if (tid == 0 && ahead < count) {
      merge_issue<KT, HV>(dn, (it + MERGE_STAGES - 1) % MERGE_STAGES, smem, bars, hdr, k0, v0, k1, v1);
      if (ahead + gridDim.x < count) dn = desc[ahead + gridDim.x];
    }
    mbar_wait(&bars[s], (it / MERGE_STAGES) & 1u);
    const MergeHdr h = hdr[s];
    const unsigned char* st = smem + SM::HDR + s * SM::STAGE;
    const K* A = reinterpret_cast<const K*>(st) + h.a_base;
    const K* B = reinterpret_cast<const K*>(st) + h.b_base;
    const uint32_t* VA = reinterpret_cast<const uint32_t*>(st + SM::KB) + h.va_base;
    const uint32_t* VB = reinterpret_cast<const uint32_t*>(st + SM::KB) + h.vb_base;
    const uint32_t base = (h.lo / tout) * tout;
    const uint32_t start = base + tid * MERGE_K;
    if (start < h.hi && start + MERGE_K > h.lo) {
      const uint32_t qs = max(start, h.lo), qe = min(start + MERGE_K, h.hi);
      const uint32_t d = qs - h.lo;
      const K* SK = reinterpret_cast<const K*>(st);
      const uint32_t* SV = reinterpret_cast<const uint32_t*>(st + SM::KB);
      K* dk = h.par ? k1 : k0;
      uint32_t* dv = h.par ? v1 : v0;
      if (qs == start && qe == start + MERGE_K) {
        // full chunk: branch-free serial merge over absolute stage indices;
        // reading one past a side stays inside the stage buffer (slack)
        const uint32_t l = corank<KT>(A, h.nA, B, h.nB, d);
        uint32_t ia = h.a_base + l, ib = h.b_base + d - l;
        const uint32_t ea = h.a_base + h.nA, eb = h.b_base + h.nB;
        const int32_t dA = (int32_t)h.va_base - (int32_t)h.a_base;
        const int32_t dB = (int32_t)h.vb_base - (int32_t)h.b_base;
        K ka = SK[ia], kb = SK[ib];
        K rk[MERGE_K];
        uint32_t ri[MERGE_K];
#pragma unroll
        for (int q = 0; q < (int)MERGE_K; ++q) {
          const bool pa = ib >= eb || (ia < ea && T::ord(ka) <= T::ord(kb));
          rk[q] = pa ? ka : kb;
          ri[q] = pa ? (uint32_t)((int32_t)ia + dA) : (uint32_t)((int32_t)ib + dB);
          ia += pa ? 1u : 0u;
          ib += pa ? 0u : 1u;
          const K nx = SK[pa ? ia : ib];
          ka = pa ? nx : ka;
          kb = pa ? kb : nx;
        }
        store_vec8<K>(dk + start, rk);
        if (HV) {
          uint32_t rv[MERGE_K];
#pragma unroll
          for (int q = 0; q < (int)MERGE_K; ++q) rv[q] = SV[ri[q]];
          store_vec8<uint32_t>(dv + start, rv);
        }
      } else {  // tile edge: the chunk is partly outside [lo, hi)
        uint32_t ia = corank<KT>(A, h.nA, B, h.nB, d), ib = d - ia;
#pragma unroll
        for (int q = 0; q < (int)MERGE_K; ++q) {
          const uint32_t pos = start + q;
          if (pos >= qs && pos < qe) {
            const bool takeA = ib >= h.nB || (ia < h.nA && T::ord(A[ia]) <= T::ord(B[ib]));
            if (takeA) { dk[pos] = A[ia]; if (HV) dv[pos] = VA[ia]; ++ia; }
            else { dk[pos] = B[ib]; if (HV) dv[pos] = VB[ib]; ++ib; }
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace vmps
