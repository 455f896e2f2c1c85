// engine4.cuh -- two-level fused level merges.
//
// Only non-fused nodes at even depth are materialized.  A materialized node X
// (depth d) merges its grandchildren directly: each child is either a leaf /
// fused unit (materialized) or a non-fused node at odd depth (virtual), whose
// two children are materialized.  So X's segment [i, k) in the source buffer
// holds up to four adjacent sorted runs W0 W1 | W2 W3 (W1 / W3 empty when the
// child is not split), and X's output is their stable merge with ties in run
// order -- exactly Alg. 1's two merges (ties to the left run), one HBM
// pass instead of two.  Buffers: an item at depth t lives in buffer
// (t even ? t/2 : 1 + (t-1)/2) mod 2... precisely buf(t) below; every
// materialized node then reads its inputs from one buffer and writes the other.
//
// Tiles come from sampling: every G4-th element of every run is a tile
// boundary.  For a sample s of run j with key v, the number of elements of run
// i that precede it in the stable order is upper_bound(run i, v) for i < j,
// lower_bound(run i, v) for i > j, and its own index for i = j; their sum is
// its output rank.  Between consecutive samples each run contributes at most
// G4 elements, so a tile holds at most 4 G4 elements.
#pragma once
#include "engine.cuh"
#include "plan.cuh"

namespace vmps {

constexpr uint32_t G4 = 1022;  // 4 G4 + 7 <= 4096: an 8-aligned cover fits 512 x 8 outputs

__host__ __device__ __forceinline__ uint32_t buf2(uint32_t t) {
  return (t & 1u) ? (1u - (((t - 1u) >> 1) & 1u)) : ((t >> 1) & 1u);
}

struct NodeRuns {
  uint32_t b[5];  // run boundaries: W_r = [b[r], b[r+1]), b[0] = i, b[4] = k
  uint32_t par;   // output buffer
  uint32_t soff;  // first sample (tile) of the node within the level
  uint32_t pad;
};

struct TileDesc4 {
  uint32_t x;     // node (local index in the level)
  uint32_t rank;  // output rank of the tile start within the node
  uint32_t c[4];  // elements of each run before the tile
};

__device__ __forceinline__ uint32_t runs_samples(const NodeRuns& R, uint32_t g4) {
  uint32_t c = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) c += (R.b[r + 1] - R.b[r] + g4 - 1) / g4;
  return c;
}

// Children of non-fused nodes (only non-fused children are recorded).
__global__ void k_child_map(const uint32_t* __restrict__ rs, const uint32_t* scalars,
                            const uint32_t* __restrict__ seg_l, const uint32_t* __restrict__ seg_r,
                            const uint32_t* __restrict__ parent, uint32_t fuse_z,
                            uint32_t* __restrict__ lchild, uint32_t* __restrict__ rchild) {
  const uint32_t r = scalars[SC_RUNS];
  for (uint32_t t = 1 + blockIdx.x * blockDim.x + threadIdx.x; t < r; t += gridDim.x * blockDim.x) {
    if (seg_size(rs, seg_l, seg_r, t) <= fuse_z) continue;
    const uint32_t P = parent[t];
    if (!P) continue;
    if (t < P) lchild[P] = t;
    else rchild[P] = t;
  }
}

// Runs and sample counts of the level's materialized nodes (zero tail to cap).
__global__ void k4_node_runs(const uint32_t* __restrict__ rs, const uint32_t* __restrict__ seg_l,
                             const uint32_t* __restrict__ seg_r, const uint32_t* __restrict__ dep,
                             const uint32_t* __restrict__ lchild, const uint32_t* __restrict__ rchild,
                             const uint32_t* __restrict__ lnodes, const uint32_t* __restrict__ level_start, int p,
                             uint32_t cap, uint32_t g4, NodeRuns* __restrict__ nr, uint32_t* __restrict__ cnt) {
  const uint32_t ls = level_start[p], m = level_start[p + 1] - ls;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= cap; x += gridDim.x * blockDim.x) {
    uint32_t c = 0;
    if (x < m) {
      const uint32_t t = lnodes[ls + x];
      NodeRuns R;
      const uint32_t i = rs[seg_l[t]], j = rs[t], k = rs[seg_r[t]];
      const uint32_t u = lchild[t], v = rchild[t];
      R.b[0] = i;
      R.b[1] = u ? rs[u] : j;
      R.b[2] = j;
      R.b[3] = v ? rs[v] : k;
      R.b[4] = k;
      R.par = buf2(dep[t] & 0xFFFFu);
      R.soff = 0;
      R.pad = 0;
      nr[x] = R;
      c = runs_samples(R, g4);
    }
    cnt[x] = c;
  }
}

template <int KT>
__device__ __forceinline__ uint32_t lower_bound_img(const typename KeyTraits<KT>::K* a, uint32_t n,
                                                    typename KeyTraits<KT>::O v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) { uint32_t m = (lo + hi) >> 1; if (KeyTraits<KT>::ord(a[m]) < v) lo = m + 1; else hi = m; }
  return lo;
}
template <int KT>
__device__ __forceinline__ uint32_t upper_bound_img(const typename KeyTraits<KT>::K* a, uint32_t n,
                                                    typename KeyTraits<KT>::O v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) { uint32_t m = (lo + hi) >> 1; if (KeyTraits<KT>::ord(a[m]) <= v) lo = m + 1; else hi = m; }
  return lo;
}

// Locate sample s of the level: node x (by the sample offsets), run r, index q.
__device__ __forceinline__ void locate_sample(const uint32_t* soff, uint32_t m, const NodeRuns* nr, uint32_t s,
                                              uint32_t g4, uint32_t* x, uint32_t* r, uint32_t* q) {
  uint32_t a = 0, b = m;  // last node with soff[x] <= s
  while (b - a > 1) { uint32_t mm = (a + b) >> 1; if (soff[mm] <= s) a = mm; else b = mm; }
  *x = a;
  uint32_t loc = s - soff[a];
  const NodeRuns R = nr[a];
  uint32_t rr = 0;
  for (; rr < 4; ++rr) {
    const uint32_t ns = (R.b[rr + 1] - R.b[rr] + g4 - 1) / g4;
    if (loc < ns) break;
    loc -= ns;
  }
  *r = rr;
  *q = loc * g4;
}

// Ranks and per-run split counts of every sample of the level.
template <int KT>
__global__ void __launch_bounds__(256) k4_samples(const typename KeyTraits<KT>::K* __restrict__ k0,
                                                  const typename KeyTraits<KT>::K* __restrict__ k1,
                                                  const NodeRuns* __restrict__ nr, const uint32_t* __restrict__ soff,
                                                  const uint32_t* __restrict__ level_start, int p, uint32_t g4,
                                                  uint32_t* __restrict__ srank, uint4* __restrict__ sc) {
  using T = KeyTraits<KT>;
  const uint32_t m = level_start[p + 1] - level_start[p];
  const uint32_t total = soff[m];
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < total; s += gridDim.x * blockDim.x) {
    uint32_t x, r, q;
    locate_sample(soff, m, nr, s, g4, &x, &r, &q);
    const NodeRuns R = nr[x];
    const auto* src = R.par ? k0 : k1;  // inputs live in the other buffer
    const typename T::O v = T::ord(src[R.b[r] + q]);
    uint32_t c[4], rank = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t len = R.b[i + 1] - R.b[i];
      uint32_t ci;
      if (i < (int)r) ci = upper_bound_img<KT>(src + R.b[i], len, v);
      else if (i > (int)r) ci = lower_bound_img<KT>(src + R.b[i], len, v);
      else ci = q;
      c[i] = ci;
      rank += ci;
    }
    srank[s] = rank;
    sc[s] = make_uint4(c[0], c[1], c[2], c[3]);
  }
}

// Sorted position of every sample within its node -> the tile list.
__global__ void __launch_bounds__(256) k4_order(const NodeRuns* __restrict__ nr, const uint32_t* __restrict__ soff,
                                                const uint32_t* __restrict__ level_start, int p, uint32_t g4,
                                                const uint32_t* __restrict__ srank, const uint4* __restrict__ sc,
                                                TileDesc4* __restrict__ tiles) {
  const uint32_t m = level_start[p + 1] - level_start[p];
  const uint32_t total = soff[m];
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < total; s += gridDim.x * blockDim.x) {
    uint32_t x, r, q;
    locate_sample(soff, m, nr, s, g4, &x, &r, &q);
    const NodeRuns R = nr[x];
    const uint32_t rank = srank[s];
    uint32_t pos = q / g4, base = soff[x];
    for (uint32_t i = 0; i < 4; ++i) {
      const uint32_t ns = (R.b[i + 1] - R.b[i] + g4 - 1) / g4;
      if (i != r && ns) {  // samples of run i with a smaller rank (ranks increase within a run)
        uint32_t lo = 0, hi = ns;
        while (lo < hi) { uint32_t mm = (lo + hi) >> 1; if (srank[base + mm] < rank) lo = mm + 1; else hi = mm; }
        pos += lo;
      }
      base += ns;
    }
    TileDesc4 d;
    d.x = x;
    d.rank = rank;
    const uint4 c = sc[s];
    d.c[0] = c.x; d.c[1] = c.y; d.c[2] = c.z; d.c[3] = c.w;
    tiles[soff[x] + pos] = d;
  }
}

// ---------------------------------------------------------------------------
// The fused merge: persistent CTAs, 2-stage TMA pipeline of 4+4 windows.
// ---------------------------------------------------------------------------
template <int KT, bool HV>
struct Merge4Smem {
  using K = typename KeyTraits<KT>::K;
  static constexpr uint32_t KB = 4096 * sizeof(K) + 256;
  static constexpr uint32_t VB = HV ? 4096 * 4 + 256 : 0;
  static constexpr uint32_t STAGE = KB + VB;
  static constexpr uint32_t HDR = 512;
  static constexpr uint32_t IK = 4096 * sizeof(K);  // intermediate keys
  static constexpr uint32_t II = 4096 * 2;          // intermediate value indices (u16)
  static constexpr uint32_t BYTES = HDR + 2 * STAGE + IK + II;
};

struct Merge4Hdr {
  uint32_t kb[4], n[4];  // key element offset / count of each window in the stage
  uint32_t vb[4];        // value element offset of each window
  uint32_t lo, hi, par, pad;
};
static_assert(64 + 2 * sizeof(Merge4Hdr) <= 512, "merge4 header area");

template <int KT, bool HV>
__device__ __forceinline__ void merge4_issue(const TileDesc4& d, const TileDesc4* dn_or_null, const NodeRuns& R,
                                             uint32_t s, unsigned char* smem, uint64_t* bars, Merge4Hdr* hdr,
                                             const typename KeyTraits<KT>::K* k0, const uint32_t* v0,
                                             const typename KeyTraits<KT>::K* k1, const uint32_t* v1) {
  using SM = Merge4Smem<KT, HV>;
  using K = typename KeyTraits<KT>::K;
  const K* sk = R.par ? k0 : k1;
  const uint32_t* sv = R.par ? v0 : v1;
  uint32_t c1[4];
  uint32_t rank1;
  if (dn_or_null) {
#pragma unroll
    for (int i = 0; i < 4; ++i) c1[i] = dn_or_null->c[i];
    rank1 = dn_or_null->rank;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) c1[i] = R.b[i + 1] - R.b[i];
    rank1 = R.b[4] - R.b[0];
  }
  unsigned char* st = smem + SM::HDR + s * SM::STAGE;
  Merge4Hdr h;
  uint32_t koff = 0, voff = 0, total = 0;
  uintptr_t kg[4], vg[4];
  uint32_t kbytes[4], vbytes[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t n = c1[i] - d.c[i];
    const uint32_t off = R.b[i] + d.c[i];
    const uintptr_t ga = (uintptr_t)(sk + off), ga0 = ga & ~(uintptr_t)15;
    const uint32_t bk = n ? (uint32_t)(((ga + (uintptr_t)n * sizeof(K) + 15) & ~(uintptr_t)15) - ga0) : 0u;
    h.kb[i] = (koff + (uint32_t)(ga - ga0)) / sizeof(K);
    h.n[i] = n;
    kg[i] = ga0;
    kbytes[i] = bk;
    koff += bk;
    if (HV) {
      const uintptr_t va = (uintptr_t)(sv + off), va0 = va & ~(uintptr_t)15;
      const uint32_t bv = n ? (uint32_t)(((va + (uintptr_t)n * 4 + 15) & ~(uintptr_t)15) - va0) : 0u;
      h.vb[i] = (voff + (uint32_t)(va - va0)) / 4;
      vg[i] = va0;
      vbytes[i] = bv;
      voff += bv;
    } else {
      h.vb[i] = 0;
    }
    total += kbytes[i] + (HV ? vbytes[i] : 0u);
  }
  h.lo = R.b[0] + d.rank;
  h.hi = R.b[0] + rank1;
  h.par = R.par;
  h.pad = 0;
  hdr[s] = h;
  mbar_arrive_expect_tx(&bars[s], total);
  uint32_t o = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (kbytes[i]) bulk_g2s(st + o, (const void*)kg[i], kbytes[i], &bars[s]);
    o += kbytes[i];
  }
  if (HV) {
    o = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (vbytes[i]) bulk_g2s(st + SM::KB + o, (const void*)vg[i], vbytes[i], &bars[s]);
      o += vbytes[i];
    }
  }
}

// Merge-path co-rank over two shared-memory sequences (ties to A).
template <int KT>
__device__ __forceinline__ uint32_t corank_s(const typename KeyTraits<KT>::K* A, uint32_t nA,
                                             const typename KeyTraits<KT>::K* B, uint32_t nB, uint32_t d) {
  return corank<KT>(A, nA, B, nB, d);
}

// Step A: P01 = W0 (+) W1 into [0, n01), P23 = W2 (+) W3 into [n01, T4) of
// the intermediate, KQ outputs per thread; each entry keeps the stage index of
// its value.  A chunk straddling n01 is split into its two sub-merges.
template <int KT, int KQ>
__device__ __forceinline__ void merge4_stepA(const typename KeyTraits<KT>::K* SK, const Merge4Hdr& h,
                                             uint32_t n01, uint32_t T4, typename KeyTraits<KT>::K* IKs,
                                             uint16_t* IIs) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  const uint32_t q0 = threadIdx.x * KQ, q1 = min(q0 + (uint32_t)KQ, T4);
  uint32_t q = q0;
  while (q < q1) {
    const bool first = q < n01;
    const uint32_t e = first ? min(q1, n01) : q1;
    const uint32_t wa = first ? 0u : 2u;
    const K* A = SK + h.kb[wa];
    const K* B = SK + h.kb[wa + 1];
    const uint32_t nA = h.n[wa], nB = h.n[wa + 1];
    const uint32_t d0 = first ? q : q - n01;
    uint32_t ia = corank<KT>(A, nA, B, nB, d0), ib = d0 - ia;
    K ka = A[min(ia, nA ? nA - 1 : 0u)], kb = B[min(ib, nB ? nB - 1 : 0u)];
    for (; q < e; ++q) {
      const bool pa = ib >= nB || (ia < nA && T::ord(ka) <= T::ord(kb));
      IKs[q] = pa ? ka : kb;
      IIs[q] = (uint16_t)(pa ? h.vb[wa] + ia : h.vb[wa + 1] + ib);
      ia += pa ? 1u : 0u;
      ib += pa ? 0u : 1u;
      if (pa) { if (ia < nA) ka = A[ia]; }
      else { if (ib < nB) kb = B[ib]; }
    }
  }
}

template <int KQ>
__device__ __forceinline__ void store_chunk(uint32_t* dst, const uint32_t (&r)[8]) {
  if (KQ == 8) { st_v4(dst, r[0], r[1], r[2], r[3]); st_v4(dst + 4, r[4], r[5], r[6], r[7]); }
  else if (KQ == 4) st_v4(dst, r[0], r[1], r[2], r[3]);
  else { dst[0] = r[0]; dst[1] = r[1]; }
}
template <int KQ>
__device__ __forceinline__ void store_chunk(uint64_t* dst, const uint64_t (&r)[8]) {
#pragma unroll
  for (int q = 0; q < KQ; q += 2)
    st_v4(dst + q, (uint32_t)r[q], (uint32_t)(r[q] >> 32), (uint32_t)r[q + 1], (uint32_t)(r[q + 1] >> 32));
}

// Step B: output = P01 (+) P23 for KQ-aligned chunks of global positions.
template <int KT, bool HV, int KQ>
__device__ __forceinline__ void merge4_stepB(const typename KeyTraits<KT>::K* IKs, const uint16_t* IIs,
                                             const uint32_t* SV, const Merge4Hdr& h, uint32_t n01, uint32_t T4,
                                             typename KeyTraits<KT>::K* k0, uint32_t* v0,
                                             typename KeyTraits<KT>::K* k1, uint32_t* v1) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  const uint32_t start = (h.lo & ~(uint32_t)(KQ - 1)) + threadIdx.x * KQ;
  if (!(start < h.hi && start + KQ > h.lo)) return;
  const uint32_t qs = max(start, h.lo), qe = min(start + (uint32_t)KQ, h.hi);
  const uint32_t d = qs - h.lo;
  const uint32_t nA = n01, nB = T4 - n01;
  const K* A = IKs;
  const K* B = IKs + n01;
  uint32_t ia = corank<KT>(A, nA, B, nB, d), ib = d - ia;
  // carried heads; a read one past a side stays inside the intermediate
  K ka = IKs[min(ia, T4 - 1)], kb = IKs[min(n01 + ib, T4 - 1)];
  K rk[8];
  uint32_t ri[8], rv[8];
#pragma unroll
  for (int q = 0; q < KQ; ++q) {
    const uint32_t pos = start + q;
    if (pos >= qs && pos < qe) {
      const bool pa = ib >= nB || (ia < nA && T::ord(ka) <= T::ord(kb));
      rk[q] = pa ? ka : kb;
      ri[q] = pa ? ia : nA + ib;
      ia += pa ? 1u : 0u;
      ib += pa ? 0u : 1u;
      const K nx = IKs[min(pa ? ia : nA + ib, T4 - 1)];
      ka = pa ? nx : ka;
      kb = pa ? kb : nx;
    } else {
      rk[q] = K(0);
      ri[q] = 0;
    }
  }
  if (HV) {
#pragma unroll
    for (int q = 0; q < KQ; ++q) rv[q] = SV[IIs[ri[q]]];
  }
  K* dk = h.par ? k1 : k0;
  uint32_t* dv = h.par ? v1 : v0;
  if (qs == start && qe == start + KQ) {
    store_chunk<KQ>(dk + start, rk);
    if (HV) store_chunk<KQ>(dv + start, rv);
  } else {
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const uint32_t pos = start + q;
      if (pos >= qs && pos < qe) { dk[pos] = rk[q]; if (HV) dv[pos] = rv[q]; }
    }
  }
}

template <int KT, bool HV>
__global__ void __launch_bounds__(MERGE_BLOCK, 2) k4_merge_level(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const TileDesc4* __restrict__ tiles, const NodeRuns* __restrict__ nr, const uint32_t* __restrict__ soff,
    const uint32_t* __restrict__ level_start, int p) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  using SM = Merge4Smem<KT, HV>;
  static_assert(MERGE_BLOCK * MERGE_K == 4096, "merge4 tile");
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  Merge4Hdr* hdr = reinterpret_cast<Merge4Hdr*>(smem + 64);
  K* IKs = reinterpret_cast<K*>(smem + SM::HDR + 2 * SM::STAGE);
  uint16_t* IIs = reinterpret_cast<uint16_t*>(smem + SM::HDR + 2 * SM::STAGE + SM::IK);
  const uint32_t m = level_start[p + 1] - level_start[p];
  const uint32_t count = soff[m];
  if (blockIdx.x >= count) return;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t tau, uint32_t s) {
    const TileDesc4 d = tiles[tau];
    const bool more = tau + 1 < count;
    TileDesc4 dn;
    if (more) dn = tiles[tau + 1];
    const bool same = more && dn.x == d.x;
    merge4_issue<KT, HV>(d, same ? &dn : nullptr, nr[d.x], s, smem, bars, hdr, k0, v0, k1, v1);
  };
  if (tid == 0) issue(blockIdx.x, 0);
  uint32_t it = 0;
  for (uint32_t tau = blockIdx.x; tau < count; tau += gridDim.x, ++it) {
    const uint32_t s = it & 1u;
    if (tid == 0 && tau + gridDim.x < count) issue(tau + gridDim.x, s ^ 1u);
    mbar_wait(&bars[s], (it >> 1) & 1u);
    const Merge4Hdr h = hdr[s];
    const unsigned char* st = smem + SM::HDR + s * SM::STAGE;
    const K* SK = reinterpret_cast<const K*>(st);
    const uint32_t* SV = reinterpret_cast<const uint32_t*>(st + SM::KB);
    const uint32_t n01 = h.n[0] + h.n[1], T4 = h.hi - h.lo;
    // outputs per thread chosen per tile so every warp has work
    const uint32_t kq = T4 <= 1020 ? 2u : (T4 <= 2040 ? 4u : 8u);
    if (kq == 2) merge4_stepA<KT, 2>(SK, h, n01, T4, IKs, IIs);
    else if (kq == 4) merge4_stepA<KT, 4>(SK, h, n01, T4, IKs, IIs);
    else merge4_stepA<KT, 8>(SK, h, n01, T4, IKs, IIs);
    __syncthreads();
    if (kq == 2) merge4_stepB<KT, HV, 2>(IKs, IIs, SV, h, n01, T4, k0, v0, k1, v1);
    else if (kq == 4) merge4_stepB<KT, HV, 4>(IKs, IIs, SV, h, n01, T4, k0, v0, k1, v1);
    else merge4_stepB<KT, HV, 8>(IKs, IIs, SV, h, n01, T4, k0, v0, k1, v1);
    __syncthreads();
  }
}

}  // namespace vmps
