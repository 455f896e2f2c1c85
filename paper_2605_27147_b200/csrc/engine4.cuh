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
// Tiles are aligned output windows of T = 4096 positions, like the one-level
// engine; their exact 4-way splits come from a nested merge-path search
// (corank4 below), so every interior tile merges exactly T outputs.
#pragma once
#include "engine.cuh"
#include "plan.cuh"

namespace vmps {

__host__ __device__ __forceinline__ uint32_t buf2(uint32_t t) {
  return (t & 1u) ? (1u - (((t - 1u) >> 1) & 1u)) : ((t >> 1) & 1u);
}

struct NodeRuns {
  uint32_t b[5];  // run boundaries: W_r = [b[r], b[r+1]), b[0] = i, b[4] = k
  uint32_t par;   // output buffer
  uint32_t pad[2];
};

// Threads of the 4-way merge.  Steps A and B give each thread KA = 9
// consecutive outputs: an odd chunk length makes the threads' co-rank probes
// and merge heads (about KA t / 2 apart) and their intermediate / staging
// writes (KA t apart) fall into distinct shared-memory banks -- with 8 they
// sat 4 and 8 words apart, 4- and 8-way conflicts on the pipe that bounds
// this kernel (l1tex data-pipe wavefronts ~88% busy, profiles/).  Copy and
// two-run tiles keep 8-output chunks stored straight to global memory (they
// are output-aligned, 128-bit stores).  17 consumer warps cover both:
// 4096 / 8 = 512 chunks, and up to ceil(n01 / 9) + ceil(n23 / 9) <= 457.
constexpr int M4_KQ = 8;                       // copy / two-run tiles
#ifndef VMPS_M4_KA
#define VMPS_M4_KA 9
#endif
constexpr uint32_t M4_KA = VMPS_M4_KA;         // steps A and B (odd)
#ifndef VMPS_M4_IV
#define VMPS_M4_IV 1
#endif
constexpr bool M4_IV = VMPS_M4_IV;             // step A carries the payload (see Merge4Smem)
#ifndef VMPS_M4_PF
#define VMPS_M4_PF 1
#endif
constexpr bool M4_PF = VMPS_M4_PF;             // merge_serial with one-ahead prefetch
#ifndef VMPS_M4_EVICT_FIRST
#define VMPS_M4_EVICT_FIRST 1
#endif
constexpr bool M4_EVICT_FIRST = VMPS_M4_EVICT_FIRST;  // 4-byte keys: the level merge's bulk loads evict-first in L2
constexpr uint32_t M4_NT = 4096 / M4_KQ + 32;  // consumer threads (17 warps)
constexpr uint32_t M4_THREADS = M4_NT + 32;    // + the producer warp
static_assert((4096 + M4_KA - 1) / M4_KA + 1 <= M4_NT, "step A chunks");

struct TileDesc4 {
  uint32_t x;     // node (local index in the level)
  uint32_t rank;  // output rank of the tile start within the node
  uint32_t c[4];  // elements of each run before the tile
};

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

// Runs of the level's materialized nodes.
__global__ void k4_node_runs(const uint32_t* __restrict__ rs, const uint32_t* __restrict__ seg_l,
                             const uint32_t* __restrict__ seg_r, const uint32_t* __restrict__ dep,
                             const uint32_t* __restrict__ lchild, const uint32_t* __restrict__ rchild,
                             const uint32_t* __restrict__ lnodes, const uint32_t* __restrict__ level_start, int p,
                             NodeRuns* __restrict__ nr) {
  const uint32_t ls = level_start[p], m = level_start[p + 1] - ls;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < m; x += gridDim.x * blockDim.x) {
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
    R.pad[0] = R.pad[1] = 0;
    nr[x] = R;
  }
}

// ---------------------------------------------------------------------------
// Exact 4-way co-ranks at aligned output positions.
//
// X = merge(L, R), L = merge(W0, W1), R = merge(W2, W3), ties to the left at
// both levels (Alg. 2), i.e. the stable merge of W0 W1 W2 W3.  For an
// output diagonal d of X the split (c0, c1, c2, c3) is found by the outer
// merge-path search over a = #L among the first d outputs, where L[a] and
// R[d-a-1] come from inner merge-path co-ranks.  Every inner search is
// bracketed by the co-ranks already evaluated (co-ranks are monotone and grow
// by at most the diagonal step), so the brackets shrink with the outer window.
// ---------------------------------------------------------------------------
template <int KT>
struct InnerCR {
  using K = typename KeyTraits<KT>::K;
  const K* A;
  const K* B;
  uint32_t nA, nB;
  uint32_t xl, cl, xh, ch;  // known co-ranks c(xl) = cl <= c(x) <= c(xh) = ch
  __device__ __forceinline__ void init(const K* a, uint32_t na, const K* b, uint32_t nb) {
    A = a; B = b; nA = na; nB = nb;
    xl = 0; cl = 0; xh = na + nb; ch = na;
  }
  // co-rank at x (xl <= x <= xh): #A among the first x outputs of merge(A, B)
  __device__ __forceinline__ uint32_t co(uint32_t x) const {
    uint32_t lo = max(cl, ch > xh - x ? ch - (xh - x) : 0u);
    uint32_t hi = min(ch, cl + (x - xl));
    lo = max(lo, x > nB ? x - nB : 0u);
    hi = min(hi, min(x, nA));
    return corank_in<KT>(A, nA, B, nB, x, lo, hi);
  }
  // element of rank x (x < nA + nB) given c = co(x)
  __device__ __forceinline__ K elem(uint32_t x, uint32_t c) const {
    using T = KeyTraits<KT>;
    if (c < nA && (x - c >= nB || T::ord(A[c]) <= T::ord(B[x - c]))) return A[c];
    return B[x - c];
  }
  __device__ __forceinline__ void know_low(uint32_t x, uint32_t c) { xl = x; cl = c; }
  __device__ __forceinline__ void know_high(uint32_t x, uint32_t c) { xh = x; ch = c; }
  // search bounds of co(x)
  __device__ __forceinline__ void bounds(uint32_t x, uint32_t* lo, uint32_t* hi) const {
    uint32_t l = max(cl, ch > xh - x ? ch - (xh - x) : 0u);
    uint32_t h = min(ch, cl + (x - xl));
    *lo = max(l, x > nB ? x - nB : 0u);
    *hi = min(h, min(x, nA));
  }
};

#ifndef VMPS_DESC4_INTERP
#define VMPS_DESC4_INTERP 1
#endif
constexpr bool DESC4_INTERP = VMPS_DESC4_INTERP;  // regula falsi steps in the outer search
// co(x) of L and co(y) of R as one interleaved loop: the two binary searches
// are independent, so their probes overlap (half the dependent latency).
// (Regula falsi here too measured slower: cfg5 partition 5.0 -> 8.1 ms --
// the known points already bracket these searches tightly, and the two
// bisection probes it needs first plus the extra registers cost more.)
template <int KT>
__device__ __forceinline__ void co_pair(const InnerCR<KT>& L, uint32_t x, const InnerCR<KT>& R, uint32_t y,
                                        uint32_t* cx, uint32_t* cy) {
  using T = KeyTraits<KT>;
  uint32_t la, ha, lb, hb;
  L.bounds(x, &la, &ha);
  R.bounds(y, &lb, &hb);
  while (la < ha || lb < hb) {
    const uint32_t ma = (la + ha) >> 1, mb = (lb + hb) >> 1;
    const bool ga = la < ha, gb = lb < hb;
    bool pa = false, pb = false;
    if (ga) pa = T::ord(L.A[ma]) <= T::ord(L.B[x - ma - 1]);
    if (gb) pb = T::ord(R.A[mb]) <= T::ord(R.B[y - mb - 1]);
    if (ga) { if (pa) la = ma + 1; else ha = ma; }
    if (gb) { if (pb) lb = mb + 1; else hb = mb; }
  }
  *cx = la;
  *cy = lb;
}

// Split of X's first d outputs; the outer co-rank a lies in [alo, ahi]
// (caller's bound, e.g. from the previous aligned boundary).  On return c[]
// holds (c0, c1, c2, c3) and L / R know their co-ranks at a and d - a.
// hint (optional, 0xFFFFFFFF = none): an estimate of the answer; the first
// two probes then bracket [hint - HINT_W, hint + HINT_W] instead of halving,
// which narrows the outer search in two evaluations when the estimate holds
// (consecutive tiles of a node split alike) and costs two when it does not.
#ifndef VMPS_HINT_W
#define VMPS_HINT_W 96
#endif
constexpr uint32_t HINT_W = VMPS_HINT_W;
template <int KT>
__device__ __forceinline__ uint32_t corank4(InnerCR<KT>& L, InnerCR<KT>& R, uint32_t d, uint32_t alo,
                                            uint32_t ahi, uint32_t* c, uint32_t hint = 0xFFFFFFFFu,
                                            uint32_t hw = HINT_W) {
  using T = KeyTraits<KT>;
  const uint32_t nL = L.nA + L.nB, nR = R.nA + R.nB;
  // the known-low points stay valid (queries only move right: L at a >=
  // a_prev, R at d - mid - 1 >= d_prev - a_prev); reset the known-high ones
  L.know_high(nL, L.nA);
  R.know_high(nR, R.nA);
  alo = max(alo, d > nR ? d - nR : 0u);
  ahi = min(ahi, min(d, nL));
  int hint_left = hint != 0xFFFFFFFFu && ahi - alo > 4 * hw ? 2 : 0;
  // Illinois regula falsi (RFalsi) on g(m) = L[m] - R[d-m-1], g <= 0 below
  // the answer: on i.i.d. keys a few outer evaluations replace ~10
  RFalsi rf;
  rf.init();
  while (alo < ahi) {
    uint32_t mid = (alo + ahi) >> 1;
    const uint32_t w0 = ahi - alo;
    bool interp = false;
    if (hint_left) {  // the probes around the hint (kept inside [alo, ahi))
      const uint32_t p = hint_left == 2 ? (hint > alo + hw ? hint - hw : alo)
                                        : (hint + hw < ahi ? hint + hw : ahi - 1);
      mid = min(max(p, alo), ahi - 1);
      --hint_left;
    } else if (DESC4_INTERP) {
      mid = rf.probe(alo, ahi, &interp);
    }
    const uint32_t r = d - mid - 1;  // < nR since mid >= d - nR
    uint32_t cL, cR;
    co_pair<KT>(L, mid, R, r, &cL, &cR);
    const auto kL = L.elem(mid, cL), kR = R.elem(r, cR);
    const auto oL = T::ord(kL), oR = T::ord(kR);
    const double g = interp_gap<KT>(kL, kR);
    if (oL <= oR) {  // L[mid] precedes R[d-mid-1]
      alo = mid + 1;
      L.know_low(mid, cL);
      R.know_high(r, cR);
    } else {
      ahi = mid;
      L.know_high(mid, cL);
      R.know_low(r, cR);
    }
    rf.update(oL <= oR, g, w0, ahi - alo, interp);
  }
  const uint32_t a = alo;
  uint32_t c0, c2;
  co_pair<KT>(L, a, R, d - a, &c0, &c2);
  L.know_low(a, c0);
  R.know_low(d - a, c2);
  c[0] = c0; c[1] = a - c0; c[2] = c2; c[3] = d - a - c2;
  return a;
}

// The same split found by a warp: each round the 32 lanes evaluate 32
// outer candidates spread over [alo, ahi) at once (each with its own inner
// co-rank searches), a ballot finds the first candidate that fails, and the
// neighbouring lanes' inner co-ranks become the next round's known points;
// the outer range shrinks ~33x per round instead of 2x per dependent step.
// For levels of few tiles, where each thread's chain of dependent probes is
// the bound and the probe traffic is small.  All lanes return the split.
template <int KT>
__device__ __forceinline__ uint32_t corank4_warp(InnerCR<KT>& L, InnerCR<KT>& R, uint32_t d, uint32_t* c,
                                                 uint32_t lane) {
  using T = KeyTraits<KT>;
  const uint32_t nL = L.nA + L.nB, nR = R.nA + R.nB;
  uint32_t alo = d > nR ? d - nR : 0u, ahi = min(d, nL);
  // g = L[m] - R[d-m-1] at alo - 1 and at ahi once known (warp-uniform): a
  // round after the first spreads its candidates over a window of 1/32 of
  // the bracket around the interpolated crossing (regula falsi, as in
  // corank4), so a hit narrows the bracket ~1000x; a miss (all candidates on
  // one side) is followed by a uniform round
  double gT = (double)NAN, gF = (double)NAN;
  bool missed = false;
  while (alo < ahi) {
    uint32_t wl = alo, w = ahi - alo;
    bool win = false;
    if (DESC4_INTERP && w >= 256u && !missed && !isnan(gT) && !isnan(gF) && gF > gT) {
      const double x = (double)alo - 1.0 + (-gT / (gF - gT)) * (double)(w + 1);
      const uint32_t cx = x <= (double)alo ? alo : x >= (double)(ahi - 1) ? ahi - 1 : (uint32_t)x;
      const uint32_t half = max(16u, w >> 6);
      wl = cx > alo + half ? cx - half : alo;
      w = min(ahi, cx + half + 1) - wl;
      win = true;
    }
    // candidates m_l strictly increasing in [wl, wl + w) (lanes past the range idle)
    const bool act = w >= 32u || lane < w;
    const uint32_t m = w >= 32u ? wl + (uint32_t)(((uint64_t)w * lane) / 32u) : wl + lane;
    bool pr = false;
    double g = 0.0;
    uint32_t cL = 0, cR = 0;
    const uint32_t r = d - m - 1;
    if (act) {
      co_pair<KT>(L, m, R, r, &cL, &cR);
      const auto kL = L.elem(m, cL), kR = R.elem(r, cR);
      pr = T::ord(kL) <= T::ord(kR);  // L[m] precedes R[d-m-1]
      g = interp_gap<KT>(kL, kR);
    }
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, pr);
    const uint32_t nact = w >= 32u ? 32u : w;
    const uint32_t f = (uint32_t)__popc(bal);  // predicate is monotone: lanes [0, f) true
    const uint32_t mT = __shfl_sync(0xFFFFFFFFu, m, f > 0 ? f - 1 : 0);
    const uint32_t cLT = __shfl_sync(0xFFFFFFFFu, cL, f > 0 ? f - 1 : 0);
    const uint32_t cRT = __shfl_sync(0xFFFFFFFFu, cR, f > 0 ? f - 1 : 0);
    const uint32_t mF = __shfl_sync(0xFFFFFFFFu, m, f < 32u ? f : 31u);
    const uint32_t cLF = __shfl_sync(0xFFFFFFFFu, cL, f < 32u ? f : 31u);
    const uint32_t cRF = __shfl_sync(0xFFFFFFFFu, cR, f < 32u ? f : 31u);
    const double gTn = __shfl_sync(0xFFFFFFFFu, g, f > 0 ? f - 1 : 0);
    const double gFn = __shfl_sync(0xFFFFFFFFu, g, f < 32u ? f : 31u);
    if (f > 0) {
      alo = mT + 1;
      L.know_low(mT, cLT);
      R.know_high(d - mT - 1, cRT);
      gT = gTn;
    }
    if (f < nact) {
      ahi = mF;
      L.know_high(mF, cLF);
      R.know_low(d - mF - 1, cRF);
      gF = gFn;
    }
    missed = win && (f == 0 || f == nact);
  }
  const uint32_t a = alo;
  uint32_t c0, c2;
  co_pair<KT>(L, a, R, d - a, &c0, &c2);
  c[0] = c0; c[1] = a - c0; c[2] = c2; c[3] = d - a - c2;
  return a;
}

// Tile descriptors of one level of the two-level schedule: tiles aligned to
// global multiples of T (enumerated by k_level_tiles / ltiles like the
// one-level engine), DESC_CHUNK consecutive tiles per thread; the first
// boundary of a chunk is a full search, the next ones search a in
// [a_prev, a_prev + T].
#ifndef VMPS_DESC4_CHUNK
#define VMPS_DESC4_CHUNK 6
#endif
constexpr uint32_t DESC4_CHUNK = VMPS_DESC4_CHUNK;
#ifndef VMPS_DESC4_HINT
#define VMPS_DESC4_HINT 2
#endif
#ifndef VMPS_DESC4_SERIAL_MIN
#define VMPS_DESC4_SERIAL_MIN 65536
#endif
constexpr uint32_t DESC4_SERIAL_MIN = VMPS_DESC4_SERIAL_MIN;
#ifndef VMPS_DESC4_WARP
#define VMPS_DESC4_WARP 1
#endif
#ifndef VMPS_DESC4_WARP_MAX
#define VMPS_DESC4_WARP_MAX 16384
#endif
constexpr uint32_t DESC4_WARP_MAX = VMPS_DESC4_WARP_MAX;  // levels below this many tiles: a warp per tile
template <int KT>
__global__ void __launch_bounds__(256) k4_desc(const typename KeyTraits<KT>::K* __restrict__ k0,
                                               const typename KeyTraits<KT>::K* __restrict__ k1,
                                               const NodeRuns* __restrict__ nr, const uint32_t* __restrict__ ltiles,
                                               const uint32_t* __restrict__ level_start,
                                               const uint32_t* __restrict__ level_tile, int p, uint32_t tout,
                                               TileDesc4* __restrict__ tiles, uint32_t warp_max) {
  const uint32_t ls = level_start[p], le = level_start[p + 1];
  const uint32_t tb = level_tile[p], te = level_tile[p + 1];
  // chunk length: a level of few tiles is bound by the length of each
  // thread's chain of dependent probes, so every tile gets its own thread
  // (below DESC4_SERIAL_MIN tiles), then three; large levels use DESC4_CHUNK
  // (fewer full searches); measured at cfg1-5 and at the paper's n = 10^7
  const uint32_t ntl = te - tb;
  if (ntl < warp_max) return;  // k4_desc_warp's level
  const uint32_t chunk = ntl < DESC4_SERIAL_MIN ? 1u : ntl < 4u * DESC4_SERIAL_MIN ? 3u : DESC4_CHUNK;
  const uint32_t nchunks = (te - tb + chunk - 1) / chunk;
  for (uint32_t ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks; ch += gridDim.x * blockDim.x) {
    const uint32_t tau0 = tb + ch * chunk;
    uint32_t a = ls, b = le;  // last bucket x with ltiles[x] <= tau0
    while (b - a > 1) { uint32_t m = (a + b) >> 1; if (ltiles[m] <= tau0) a = m; else b = m; }
    uint32_t cur = 0xFFFFFFFFu, aprev = 0, dprev = 0, aprev2 = 0, dprev2 = 0;
    InnerCR<KT> L, R;
    NodeRuns X;
    for (uint32_t q = 0; q < chunk; ++q) {
      const uint32_t tau = tau0 + q;
      if (tau >= te) break;
      while (a + 1 < le && ltiles[a + 1] <= tau) ++a;
      if (a != cur) {
        X = nr[a - ls];
        const auto* src = X.par ? k0 : k1;  // inputs live in the other buffer
        L.init(src + X.b[0], X.b[1] - X.b[0], src + X.b[1], X.b[2] - X.b[1]);
        R.init(src + X.b[2], X.b[3] - X.b[2], src + X.b[3], X.b[4] - X.b[3]);
        cur = a;
        aprev = 0;
        dprev = 0;
        aprev2 = 0;
        dprev2 = 0;
      }
      const uint32_t i = X.b[0], k = X.b[4];
      const uint32_t g = i / tout + (tau - ltiles[a]);
      const uint32_t lo = max(i, g * tout);
      const uint32_t d = lo - i;
      uint32_t c[4];
      // estimate: the previous tile's share of L among its outputs
      const uint32_t hint = (cur == a && q > 0 && d > dprev && dprev > dprev2)
                                ? aprev + (uint32_t)(((uint64_t)(aprev - aprev2) * (d - dprev)) / (dprev - dprev2))
                                : 0xFFFFFFFFu;
      uint32_t h = VMPS_DESC4_HINT ? hint : 0xFFFFFFFFu, hw = HINT_W;
#if VMPS_DESC4_HINT >= 2
      // first tile of the node in this chunk: L's share of the node, +- 2 sqrt(d)
      // (with the regula falsi steps after the two hint probes this helps
      // structured inputs too: cfg4 6.95 -> 6.53 ms, cfg5 partition 4.75 -> 4.55)
      if (h == 0xFFFFFFFFu && d > 0) {
        const uint32_t nL = (X.b[2] - X.b[0]), nX = X.b[4] - X.b[0];
        h = (uint32_t)(((uint64_t)d * nL) / nX);
        hw = max(HINT_W, 2u * (uint32_t)sqrtf((float)d));
      }
#endif
      const uint32_t av = corank4<KT>(L, R, d, aprev, aprev + (d - dprev), c, h, hw);
      aprev2 = aprev;
      dprev2 = dprev;
      aprev = av;
      dprev = d;
      TileDesc4 D;
      D.x = a - ls;
      D.rank = d;
      D.c[0] = c[0]; D.c[1] = c[1]; D.c[2] = c[2]; D.c[3] = c[3];
      tiles[tau - tb] = D;
      (void)k;
    }
  }
}


// Small levels (fewer than warp_max tiles): one warp per tile, the split by
// corank4_warp.  Launched beside k4_desc, which skips these levels.
template <int KT>
__global__ void __launch_bounds__(256) k4_desc_warp(const typename KeyTraits<KT>::K* __restrict__ k0,
                                                    const typename KeyTraits<KT>::K* __restrict__ k1,
                                                    const NodeRuns* __restrict__ nr,
                                                    const uint32_t* __restrict__ ltiles,
                                                    const uint32_t* __restrict__ level_start,
                                                    const uint32_t* __restrict__ level_tile, int p, uint32_t tout,
                                                    TileDesc4* __restrict__ tiles, uint32_t warp_max) {
  const uint32_t ls = level_start[p], le = level_start[p + 1];
  const uint32_t tb = level_tile[p], te = level_tile[p + 1];
  const uint32_t ntl = te - tb;
  if (ntl < warp_max) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < ntl; wi += nw) {
      const uint32_t tau = tb + wi;
      uint32_t a = ls, b = le;
      while (b - a > 1) { uint32_t m = (a + b) >> 1; if (ltiles[m] <= tau) a = m; else b = m; }
      const NodeRuns X = nr[a - ls];
      const auto* src = X.par ? k0 : k1;
      InnerCR<KT> L, R;
      L.init(src + X.b[0], X.b[1] - X.b[0], src + X.b[1], X.b[2] - X.b[1]);
      R.init(src + X.b[2], X.b[3] - X.b[2], src + X.b[3], X.b[4] - X.b[3]);
      const uint32_t i = X.b[0];
      const uint32_t g = i / tout + (tau - ltiles[a]);
      const uint32_t d = max(i, g * tout) - i;
      uint32_t c[4];
      corank4_warp<KT>(L, R, d, c, lane);
      if (lane == 0) {
        TileDesc4 D;
        D.x = a - ls;
        D.rank = d;
        D.c[0] = c[0]; D.c[1] = c[1]; D.c[2] = c[2]; D.c[3] = c[3];
        tiles[tau - tb] = D;
      }
    }
    return;
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
#ifndef VMPS_U64_STAGES
#define VMPS_U64_STAGES 2
#endif
  // stages of the TMA pipeline: u64 keys with payload use VMPS_U64_STAGES
  // (one stage fits two CTAs per SM), all others two
  static constexpr uint32_t NSTG = (sizeof(K) == 8 && HV) ? VMPS_U64_STAGES : 2u;
  // the barrier area holds two full / empty pairs and the header area two Merge4Hdr
  static_assert(NSTG >= 1 && NSTG <= 2, "merge4: at most two pipeline stages");
  // intermediate: P01 at [0, n01), P23 at [n01p, n01p + n23), n01p = n01
  // rounded up to a multiple of KA (<= 4096 + 8 positions), + read-ahead slack
  static constexpr uint32_t IPOS = 4096 + 48;
  static constexpr uint32_t IK = IPOS * sizeof(K);  // intermediate keys
  // intermediate payload: with M4_IV the values themselves (u32, gathered
  // by step A next to its key loads), else the stage index of each value (u16)
  static constexpr uint32_t II = !HV ? 0u : M4_IV ? IPOS * 4 : IPOS * 2;
  // step B output staging: keys go to the tile's stage key area (free once
  // step A is done), values to the stage value area with M4_IV (step A has
  // read it) or else to OV; both then leave by TMA bulk stores
  static constexpr uint32_t OV = (HV && !M4_IV) ? 4096 * 4 + 64 : 0;
  static constexpr uint32_t BYTES = HDR + NSTG * STAGE + IK + II + OV;
};

constexpr int M4_WARPS = M4_NT / 32;  // consumer warps of a tile (17)
struct alignas(16) Merge4Hdr {
  uint32_t kb[4], n[4];  // key element offset / count of each window in the stage
  uint32_t vb[4];        // value element offset of each window
  uint32_t lo, hi, par, mode;  // mode: 0 general, 1 two runs (W0, W2), 2 + w single run w
  // step A warp boundaries (written by the producer warp once the stage has
  // landed): bnd[w] = co-rank of the 2-way merge that intermediate position
  // 256 w belongs to (P01 = W0 (+) W1 below n01, P23 = W2 (+) W3 above), at
  // that position's diagonal within its merge
  uint16_t bnd[M4_WARPS + 1];
};
static_assert(64 + 2 * sizeof(Merge4Hdr) <= 512, "merge4 header area");

// A consumer thread's copy of a tile header: four 128-bit shared-memory loads
// (broadcast) instead of a scalar load per field and use -- the header reads
// were ~5% of the shared-memory wavefronts of this LSU-bound kernel.
struct M4H {
  uint32_t kb[4], n[4], vb[4];
  uint32_t lo, hi, par, mode;
};
__device__ __forceinline__ M4H m4_load_hdr(const Merge4Hdr* hp) {
  const uint4* q = reinterpret_cast<const uint4*>(hp);
  const uint4 a = q[0], b = q[1], c = q[2], d = q[3];
  M4H h;
  h.kb[0] = a.x; h.kb[1] = a.y; h.kb[2] = a.z; h.kb[3] = a.w;
  h.n[0] = b.x; h.n[1] = b.y; h.n[2] = b.z; h.n[3] = b.w;
  h.vb[0] = c.x; h.vb[1] = c.y; h.vb[2] = c.z; h.vb[3] = c.w;
  h.lo = d.x; h.hi = d.y; h.par = d.z; h.mode = d.w;
  return h;
}

template <int KT, bool HV>
__device__ __forceinline__ void merge4_issue(const TileDesc4& d, const TileDesc4* dn_or_null, const NodeRuns& R,
                                             uint32_t s, unsigned char* smem, uint64_t* bars, Merge4Hdr* hdr,
                                             const typename KeyTraits<KT>::K* k0, const uint32_t* v0,
                                             const typename KeyTraits<KT>::K* k1, const uint32_t* v1) {
  using SM = Merge4Smem<KT, HV>;
  using K = typename KeyTraits<KT>::K;
  constexpr bool EF = M4_EVICT_FIRST && sizeof(K) == 4;  // inputs read once per pass
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
  {  // tile class, decided once by the producer
    const uint32_t nz = (h.n[0] != 0) + (h.n[1] != 0) + (h.n[2] != 0) + (h.n[3] != 0);
    h.mode = nz == 1 ? 2u + (h.n[0] ? 0u : h.n[1] ? 1u : h.n[2] ? 2u : 3u)
                     : ((h.n[1] == 0 && h.n[3] == 0) ? 1u : 0u);
  }
  hdr[s] = h;
  mbar_arrive_expect_tx(&bars[s], total);
  uint32_t o = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (kbytes[i]) bulk_g2s<EF>(st + o, (const void*)kg[i], kbytes[i], &bars[s]);
    o += kbytes[i];
  }
  if (HV) {
    o = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (vbytes[i]) bulk_g2s<EF>(st + SM::KB + o, (const void*)vg[i], vbytes[i], &bars[s]);
      o += vbytes[i];
    }
  }
}


// KQ consecutive outputs of a stable 2-way merge in shared memory, A at
// [ia, ea) and B at [ib, eb) (absolute indices into S), ties to A.
// rk = keys, ri = the index of each output in S plus dA / dB (the position
// of its value).  Reads one past a part stay inside S (padded).  (A second,
// test-free path for chunks that cannot exhaust a part measured slower:
// 68.4 vs 67.1 ms at cfg5 -- the two unrolled bodies diverge inside warps.)
template <int KT, int KQ>
__device__ __forceinline__ void merge_serial(const typename KeyTraits<KT>::K* S, uint32_t ia, uint32_t ib,
                                             uint32_t ea, uint32_t eb, int32_t dA, int32_t dB,
                                             typename KeyTraits<KT>::K (&rk)[KQ], uint32_t (&ri)[KQ]) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  if constexpr (M4_PF && KT == VMPS_KEY_U32) {
    // heads and one-ahead prefetches of both sides: the load issued at a step
    // is first needed a step later, so its latency leaves the compare ->
    // select -> load chain (reads past a part stay inside the padded buffer).
    // u32 only: with f32 (order image per compare) and u64 keys (registers)
    // it measured slower (cfg4 6.54 -> 6.88 ms, cfg3 5.49 -> 5.58 ms)
    K ka = S[ia], kb = S[ib], ka2 = S[ia + 1], kb2 = S[ib + 1];
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const bool pa = ib >= eb || (ia < ea && T::ord(ka) <= T::ord(kb));
      rk[q] = pa ? ka : kb;
      ri[q] = pa ? (uint32_t)((int32_t)ia + dA) : (uint32_t)((int32_t)ib + dB);
      ia += pa ? 1u : 0u;
      ib += pa ? 0u : 1u;
      const K nx = S[(pa ? ia : ib) + 1];
      ka = pa ? ka2 : ka;
      kb = pa ? kb : kb2;
      ka2 = pa ? nx : ka2;
      kb2 = pa ? kb2 : nx;
    }
    return;
  }
  K ka = S[ia], kb = S[ib];
  typename T::O oa = T::ord(ka), ob = T::ord(kb);  // order images, computed once per load
#pragma unroll
  for (int q = 0; q < KQ; ++q) {
    const bool pa = ib >= eb || (ia < ea && oa <= ob);
    rk[q] = pa ? ka : kb;
    ri[q] = pa ? (uint32_t)((int32_t)ia + dA) : (uint32_t)((int32_t)ib + dB);
    ia += pa ? 1u : 0u;
    ib += pa ? 0u : 1u;
    const K nx = S[pa ? ia : ib];
    const typename T::O onx = T::ord(nx);
    ka = pa ? nx : ka;
    oa = pa ? onx : oa;
    kb = pa ? kb : nx;
    ob = pa ? ob : onx;
  }
}

// Step A: P01 = W0 (+) W1 into [0, n01), P23 = W2 (+) W3 into [n01, T4) of
// the intermediate (keys + the stage index of each value), KQ outputs per
// thread.  A chunk inside one of the two merges takes the unrolled
// branch-free path over absolute stage indices (a read one past a window
// stays inside the stage: windows are padded).  The chunk holding n01 (and
// the tile's last chunk) runs each of its parts for exactly its length, so
// that thread costs about as much as the others (P23's part starts at
// diagonal 0 and needs no search).
// Step A layout: P01 = W0 (+) W1 at intermediate positions [0, n01), P23 =
// W2 (+) W3 at [n01p, n01p + n23) with n01p = n01 rounded up to a multiple of
// KA, so every thread's KA-chunk lies in one of the two merges.
__device__ __forceinline__ uint32_t m4_n01p(uint32_t n01) { return (n01 + M4_KA - 1u) / M4_KA * M4_KA; }

// The co-rank of intermediate position q (< n01p + n23) within its 2-way
// merge; one lane of the producer warp per consumer warp boundary q = 32 KA w.
template <int KT>
__device__ __forceinline__ uint32_t merge4_boundary(const typename KeyTraits<KT>::K* SK, const Merge4Hdr& h,
                                                    uint32_t q) {
  const uint32_t n01p = m4_n01p(h.n[0] + h.n[1]);
  const uint32_t wa = q < n01p ? 0u : 2u;
  return corank<KT>(SK + h.kb[wa], h.n[wa], SK + h.kb[wa + 1], h.n[wa + 1], q - (q < n01p ? 0u : n01p));
}

// Producer warp, once stage s has landed: the step A warp boundaries of a
// general tile (lane w < M4_WARPS computes boundary w).
template <int KT>
__device__ __forceinline__ void merge4_bnds(const typename KeyTraits<KT>::K* SK, Merge4Hdr* hs, uint32_t lane) {
  const Merge4Hdr& h = *hs;
  if (h.mode != 0u || lane >= (uint32_t)M4_WARPS) return;
  const uint32_t q = lane * 32u * M4_KA;
  if (q < m4_n01p(h.n[0] + h.n[1]) + h.n[2] + h.n[3]) hs->bnd[lane] = (uint16_t)merge4_boundary<KT>(SK, h, q);
}

// Step A: P01 and P23 into the intermediate (keys + the stage index of each
// value), KA outputs per thread by the unrolled branch-free merge over
// absolute stage indices (a read past a window stays inside the stage:
// windows are padded).  A part's last chunk runs all KA steps and stores only
// its in-range outputs.  With have_bnd, the co-rank search is bracketed by the
// producer's co-ranks at this warp's boundaries.
template <int KT, bool HV>
__device__ __forceinline__ void merge4_stepA(const typename KeyTraits<KT>::K* SK, const uint32_t* SV, const M4H& h,
                                             const uint16_t* bnd, typename KeyTraits<KT>::K* IKs, void* IX,
                                             bool have_bnd) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  constexpr uint32_t KQ = M4_KA;
  const uint32_t n01 = h.n[0] + h.n[1], n23 = h.n[2] + h.n[3];
  const uint32_t n01p = m4_n01p(n01);
  const uint32_t q0 = threadIdx.x * KQ;
  const bool part0 = q0 < n01p;
  const uint32_t base = part0 ? 0u : n01p, plen = part0 ? n01 : n23;
  const uint32_t d = q0 - base;
  if (d >= plen) return;  // past P23 (part 0 chunks always start inside P01)
  const uint32_t nA = part0 ? h.n[0] : h.n[2], nB = part0 ? h.n[1] : h.n[3];
  const uint32_t ka0 = part0 ? h.kb[0] : h.kb[2], kb0 = part0 ? h.kb[1] : h.kb[3];
  const int32_t dA = (int32_t)(part0 ? h.vb[0] : h.vb[2]) - (int32_t)ka0,
                dB = (int32_t)(part0 ? h.vb[1] : h.vb[3]) - (int32_t)kb0;
  uint32_t lb = 0u, ub = 0xFFFFFFFFu;
  if (have_bnd) {
    // c(x1) = c1 <= c(d) <= c(x2) = c2, c(d) - c1 <= d - x1, c2 - c(d) <= x2 - d
    const uint32_t w = threadIdx.x >> 5;
    const uint32_t ws = w * 32u * KQ, we = ws + 32u * KQ;
    uint32_t x1 = 0u, c1 = 0u, x2 = nA + nB, c2 = nA;
    if (ws >= base) { x1 = ws - base; c1 = bnd[w]; }
    if (we < base + plen) { x2 = we - base; c2 = bnd[w + 1]; }
    lb = max(c1, c2 > x2 - d ? c2 - (x2 - d) : 0u);
    ub = min(c2, c1 + (d - x1));
  }
  const uint32_t l = corank_in<KT>(SK + ka0, nA, SK + kb0, nB, d, lb, ub);
  K rk[KQ];
  uint32_t ri[KQ];
  merge_serial<KT, (int)KQ>(SK, ka0 + l, kb0 + d - l, ka0 + nA, kb0 + nB, dA, dB, rk, ri);
  uint32_t* IVs = reinterpret_cast<uint32_t*>(IX);
  uint16_t* IIs = reinterpret_cast<uint16_t*>(IX);
  if (d + KQ <= plen) {
#pragma unroll
    for (int q = 0; q < (int)KQ; ++q) {
      IKs[q0 + q] = rk[q];
      if (HV) { if (M4_IV) IVs[q0 + q] = SV[ri[q]]; else IIs[q0 + q] = (uint16_t)ri[q]; }
    }
  } else {
#pragma unroll
    for (int q = 0; q < (int)KQ; ++q)
      if (d + q < plen) {
        IKs[q0 + q] = rk[q];
        if (HV) { if (M4_IV) IVs[q0 + q] = SV[ri[q]]; else IIs[q0 + q] = (uint16_t)ri[q]; }
      }
  }
}

template <int KQ>
__device__ __forceinline__ void store_chunk_g(uint32_t* dst, const uint32_t (&r)[KQ]) {
#pragma unroll
  for (int q = 0; q < KQ; q += 4) st_v4(dst + q, r[q], r[q + 1], r[q + 2], r[q + 3]);
}
template <int KQ>
__device__ __forceinline__ void store_chunk_g(uint64_t* dst, const uint64_t (&r)[KQ]) {
#pragma unroll
  for (int q = 0; q < KQ; q += 2)
    st_v4(dst + q, (uint32_t)r[q], (uint32_t)(r[q] >> 32), (uint32_t)r[q + 1], (uint32_t)(r[q + 1] >> 32));
}

// Elements per 16 bytes (a bulk copy's alignment unit).
template <typename X>
__host__ __device__ constexpr uint32_t vec16() { return 16u / (uint32_t)sizeof(X); }

// Step B: the tile's outputs = P01 (+) P23, KA consecutive outputs per thread
// (tile-relative positions d = KA t), written to shared staging at index
// (lo mod vec16) + d -- the stage key area for keys, OV for values -- so that
// the 16-byte aligned part of [lo, hi) is one bulk store per array.
template <int KT, bool HV>
__device__ __forceinline__ void merge4_stepB(const typename KeyTraits<KT>::K* IKs, const void* IX,
                                             const uint32_t* SV, uint32_t lo, uint32_t n01, uint32_t T4,
                                             typename KeyTraits<KT>::K* OKs, uint32_t* OVs) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  constexpr uint32_t KQ = M4_KA;
  const uint32_t d = threadIdx.x * KQ;
  const uint32_t n01p = m4_n01p(n01);  // P23 starts here (step A layout)
  const uint32_t nA = n01, nB = T4 - n01;
  // (bracketing this search by a 32-ary warp co-rank at the warp's first
  // output measured slower: cfg5 68.2 vs 67.0 ms, cfg4 7.50 vs 7.11 ms)
  if (d >= T4) return;
  const uint32_t l = corank<KT>(IKs, nA, IKs + n01p, nB, d);
  K rk[KQ];
  uint32_t ri[KQ];  // reads past the parts stay inside the intermediate (slack)
  merge_serial<KT, (int)KQ>(IKs, l, n01p + d - l, n01, n01p + nB, 0, 0, rk, ri);
  K* ok = OKs + (lo & (vec16<K>() - 1u)) + d;
  uint32_t* ov = OVs + (lo & 3u) + d;
  const uint32_t* IVs = reinterpret_cast<const uint32_t*>(IX);
  const uint16_t* IIs = reinterpret_cast<const uint16_t*>(IX);
  if (d + KQ <= T4) {
#pragma unroll
    for (int q = 0; q < (int)KQ; ++q) {
      ok[q] = rk[q];
      if (HV) ov[q] = M4_IV ? IVs[ri[q]] : SV[IIs[ri[q]]];
    }
  } else {
#pragma unroll
    for (int q = 0; q < (int)KQ; ++q)
      if (d + q < T4) {
        ok[q] = rk[q];
        if (HV) ov[q] = M4_IV ? IVs[ri[q]] : SV[IIs[ri[q]]];
      }
  }
}

// After step B (all consumers past the barrier): the staged outputs of the
// tile leave shared memory.  Thread 0 issues one bulk store per array for the
// 16-byte aligned part of [lo, hi) and waits until they have read shared
// memory; threads 32.. store the < vec16 ragged elements at either end.
template <int KT, bool HV>
__device__ __forceinline__ void merge4_flush(const typename KeyTraits<KT>::K* OKs, const uint32_t* OVs,
                                             uint32_t lo, uint32_t hi, typename KeyTraits<KT>::K* dk,
                                             uint32_t* dv) {
  using K = typename KeyTraits<KT>::K;
  constexpr uint32_t VK = vec16<K>(), VV = 4u;
  const uint32_t tid = threadIdx.x;
  const uint32_t lok = (lo + VK - 1u) & ~(VK - 1u), hik = max(hi & ~(VK - 1u), lok);
  const uint32_t lov = (lo + VV - 1u) & ~(VV - 1u), hiv = max(hi & ~(VV - 1u), lov);
  const K* sk = OKs - (lo & ~(VK - 1u));  // sk[g] = output g (shared)
  const uint32_t* sv = OVs - (lo & ~(VV - 1u));
  if (tid == 0) {
    if (hik > lok) bulk_s2g(dk + lok, sk + lok, (hik - lok) * (uint32_t)sizeof(K));
    if (HV && hiv > lov) bulk_s2g(dv + lov, sv + lov, (hiv - lov) * 4u);
    bulk_commit();
  } else if (tid >= 32u && tid < 32u + 2u * VK) {  // ragged key ends: [lo, lok) and [hik, hi)
    const uint32_t j = tid - 32u;
    const uint32_t g = j < VK ? lo + j : hik + (j - VK);
    if (j < VK ? g < min(lok, hi) : g < hi) dk[g] = sk[g];
  } else if (HV && tid >= 64u && tid < 64u + 2u * VV) {  // ragged value ends
    const uint32_t j = tid - 64u;
    const uint32_t g = j < VV ? lo + j : hiv + (j - VV);
    if (j < VV ? g < min(lov, hi) : g < hi) dv[g] = sv[g];
  }
}

// A tile fed by a single window: copy it (keys and values) to the output.
template <int KT, bool HV, int KQ>
__device__ __forceinline__ void merge4_copy(const typename KeyTraits<KT>::K* SK, const uint32_t* SV, uint32_t kb,
                                            uint32_t vb, uint32_t lo, uint32_t hi, uint32_t par,
                                            typename KeyTraits<KT>::K* k0, uint32_t* v0,
                                            typename KeyTraits<KT>::K* k1, uint32_t* v1) {
  using K = typename KeyTraits<KT>::K;
  const uint32_t start = (lo & ~(uint32_t)(KQ - 1)) + threadIdx.x * KQ;
  if (!(start < hi && start + (uint32_t)KQ > lo)) return;
  K* dk = par ? k1 : k0;
  uint32_t* dv = par ? v1 : v0;
  if (start >= lo && start + (uint32_t)KQ <= hi) {
    K rk[KQ];
    uint32_t rv[KQ];
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      rk[q] = SK[kb + (start - lo) + q];
      if (HV) rv[q] = SV[vb + (start - lo) + q];
    }
    store_chunk_g<KQ>(dk + start, rk);
    if (HV) store_chunk_g<KQ>(dv + start, rv);
  } else {
    for (uint32_t pos = max(start, lo); pos < min(start + (uint32_t)KQ, hi); ++pos) {
      dk[pos] = SK[kb + (pos - lo)];
      if (HV) dv[pos] = SV[vb + (pos - lo)];
    }
  }
}

// A tile whose runs are W0 and W2 only: merge them straight from the stage
// (absolute stage indices; a read one past a window stays in the stage).
template <int KT, bool HV, int KQ>
__device__ __forceinline__ void merge4_direct(const typename KeyTraits<KT>::K* SK, const uint32_t* SV,
                                              const M4H& h, uint32_t lo, uint32_t hi, uint32_t par,
                                              typename KeyTraits<KT>::K* k0, uint32_t* v0,
                                              typename KeyTraits<KT>::K* k1, uint32_t* v1) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  const uint32_t start = (lo & ~(uint32_t)(KQ - 1)) + threadIdx.x * KQ;
  if (!(start < hi && start + (uint32_t)KQ > lo)) return;
  K* dk = par ? k1 : k0;
  uint32_t* dv = par ? v1 : v0;
  const uint32_t nA = h.n[0], nB = h.n[2];
  const uint32_t ka0 = h.kb[0], kb0 = h.kb[2];
  const int32_t dA = (int32_t)h.vb[0] - (int32_t)ka0, dB = (int32_t)h.vb[2] - (int32_t)kb0;
  const uint32_t qs = max(start, lo);
  const uint32_t d = qs - lo;
  const uint32_t l = corank<KT>(SK + ka0, nA, SK + kb0, nB, d);
  K rk[KQ];
  uint32_t ri[KQ];
  merge_serial<KT, KQ>(SK, ka0 + l, kb0 + d - l, ka0 + nA, kb0 + nB, dA, dB, rk, ri);
  if (qs == start && start + (uint32_t)KQ <= hi) {
    store_chunk_g<KQ>(dk + start, rk);
    if (HV) {
      uint32_t rv[KQ];
#pragma unroll
      for (int q = 0; q < KQ; ++q) rv[q] = SV[ri[q]];
      store_chunk_g<KQ>(dv + start, rv);
    }
  } else {
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const uint32_t pos = qs + q;
      if (pos < hi && pos < start + (uint32_t)KQ) { dk[pos] = rk[q]; if (HV) dv[pos] = SV[ri[q]]; }
    }
  }
}

// One tile on the consumer side (17 warps), shared by the level merge and
// the pull-merge.  Copy tiles and two-run tiles store 8-output chunks
// straight to global memory; general tiles run steps A and B through the
// intermediate and leave by bulk stores.  Every consumer warp arrives once on
// empty[s] when it no longer needs stage s (warp 0 only after the bulk
// stores have read the stage's key area).
template <int KT, bool HV>
__device__ __forceinline__ void merge4_tile(const Merge4Hdr* hp, unsigned char* st, typename KeyTraits<KT>::K* IKs,
                                            void* IX, uint32_t* OVa, uint64_t* empty_s, bool have_bnd,
                                            typename KeyTraits<KT>::K* k0, uint32_t* v0,
                                            typename KeyTraits<KT>::K* k1, uint32_t* v1) {
  using K = typename KeyTraits<KT>::K;
  using SM = Merge4Smem<KT, HV>;
  const uint32_t lane = threadIdx.x & 31u;
  K* SK = reinterpret_cast<K*>(st);
  const uint32_t* SV = reinterpret_cast<const uint32_t*>(st + SM::KB);
  const M4H h = m4_load_hdr(hp);
  const uint32_t lo = h.lo, hi = h.hi, par = h.par;
  const uint32_t mode = h.mode;
  if (mode >= 2) {
    // run-skip tile: every output comes from one run, so
    // the tile is a compare-free copy of that window
    const uint32_t wsrc = mode - 2;
    const uint32_t kbw = wsrc == 0 ? h.kb[0] : wsrc == 1 ? h.kb[1] : wsrc == 2 ? h.kb[2] : h.kb[3];
    const uint32_t vbw = wsrc == 0 ? h.vb[0] : wsrc == 1 ? h.vb[1] : wsrc == 2 ? h.vb[2] : h.vb[3];
    merge4_copy<KT, HV, M4_KQ>(SK, SV, kbw, vbw, lo, hi, par, k0, v0, k1, v1);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_s);
  } else if (mode == 1) {
    // both children are single runs (leaves / units): one 2-way merge
    // straight from the stage, no intermediate
    merge4_direct<KT, HV, M4_KQ>(SK, SV, h, lo, hi, par, k0, v0, k1, v1);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_s);
  } else {
    const uint32_t n01 = h.n[0] + h.n[1], T4 = hi - lo;
    merge4_stepA<KT, HV>(SK, SV, h, hp->bnd, IKs, IX, have_bnd);
    named_bar_sync(1, M4_NT);  // the intermediate is complete; the stage keys (and with M4_IV values) are dead
    uint32_t* OVs = M4_IV ? reinterpret_cast<uint32_t*>(st + SM::KB) : OVa;
    merge4_stepB<KT, HV>(IKs, IX, SV, lo, n01, T4, SK, OVs);
    fence_proxy_async_smem();  // staged outputs -> visible to the bulk stores
    named_bar_sync(1, M4_NT);  // staging complete; the intermediate is free for the next tile
    merge4_flush<KT, HV>(SK, OVs, lo, hi, par ? k1 : k0, par ? v1 : v0);
    if (threadIdx.x == 0) bulk_wait_read0();  // the stage / OV may be overwritten from here on
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_s);
  }
}

// The fused merge: persistent CTAs; 17 consumer warps merge, one producer
// warp loads descriptors and issues the bulk copies of the next tile into
// the free stage (full / empty mbarrier pairs), then computes the step A
// warp boundaries of that tile once it has landed (ready barrier).
template <int KT, bool HV, int KQ>
__global__ void __launch_bounds__(M4_THREADS, 2) k4_merge_level(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const TileDesc4* __restrict__ tiles, const NodeRuns* __restrict__ nr,
    const uint32_t* __restrict__ level_tile, int p) {
  using K = typename KeyTraits<KT>::K;
  using SM = Merge4Smem<KT, HV>;
  constexpr uint32_t NT = M4_NT;  // consumer threads
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 2;
  uint64_t* ready = full + 4;  // step A boundaries written (producer warp, 32 arrivals)
  Merge4Hdr* hdr = reinterpret_cast<Merge4Hdr*>(smem + 64);
  K* IKs = reinterpret_cast<K*>(smem + SM::HDR + SM::NSTG * SM::STAGE);
  void* IX = smem + SM::HDR + SM::NSTG * SM::STAGE + SM::IK;
  uint32_t* OVs = reinterpret_cast<uint32_t*>(smem + SM::HDR + SM::NSTG * SM::STAGE + SM::IK + SM::II);
  const uint32_t count = level_tile[p + 1] - level_tile[p];
  if (blockIdx.x >= count) return;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], NT / 32);
    mbar_init(&empty[1], NT / 32);
    mbar_init(&ready[0], 32);
    mbar_init(&ready[1], 32);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= NT) {  // producer warp
    const uint32_t plane = tid - NT;
    uint32_t it = 0;
    // the next tile's descriptors (and its node) are loaded before the wait
    // for its stage, so their latency overlaps the consumers' current tile
    TileDesc4 d, dn;
    NodeRuns R;
    bool same = false;
    auto fetch = [&](uint32_t t) {
      d = tiles[t];
      same = t + 1 < count && (dn = tiles[t + 1], dn.x == d.x);
      R = nr[d.x];
    };
    if (plane == 0) fetch(blockIdx.x);
    for (uint32_t tau = blockIdx.x; tau < count; tau += gridDim.x, ++it) {
      const uint32_t s = it % SM::NSTG;
      if (plane == 0) {
        if (it >= SM::NSTG) mbar_wait_backoff(&empty[s], ((it / SM::NSTG) - 1) & 1u);
        merge4_issue<KT, HV>(d, same ? &dn : nullptr, R, s, smem, full, hdr, k0, v0, k1, v1);
      }
      mbar_wait_backoff(&full[s], (it / SM::NSTG) & 1u);
      merge4_bnds<KT>(reinterpret_cast<const K*>(smem + SM::HDR + s * SM::STAGE), hdr + s, plane);
      mbar_arrive(&ready[s]);
      if (plane == 0 && tau + gridDim.x < count) fetch(tau + gridDim.x);
    }
    return;
  }
  uint32_t it = 0;
  for (uint32_t tau = blockIdx.x; tau < count; tau += gridDim.x, ++it) {
    const uint32_t s = it % SM::NSTG;
    mbar_wait(&ready[s], (it / SM::NSTG) & 1u);
    merge4_tile<KT, HV>(hdr + s, smem + SM::HDR + s * SM::STAGE, IKs, IX, OVs, &empty[s], true, k0, v0, k1, v1);
  }
  if (tid == 0) bulk_wait0();  // the last bulk stores are complete before the kernel ends
}

}  // namespace vmps

namespace vmps {
// ---------------------------------------------------------------------------
// Pull-merge: the stable merge of up to four sorted pieces
// that live at four arbitrary device addresses -- on a multi-GPU box, the
// co-ranked pieces of the other ranks' shards, read through peer mappings
// (CUDA IPC over NVLink) -- written once into one output array.  It replaces
// "all-to-all into a receive buffer, then merge the buffer": the pieces are
// read straight from where they are, by the same TMA-staged 4-way engine.
// Ties go to the lower piece index (the lower source rank).
// ---------------------------------------------------------------------------
template <int KT>
struct PullSrc {
  const typename KeyTraits<KT>::K* kp[4];
  const uint32_t* vp[4];
  uint32_t n[4];
  uint32_t N;     // sum of n[]
  uint32_t base;  // output position of the merge's first element (tiles align to global multiples of 4096)
};

// Tile descriptors at output positions base + d aligned to global multiples
// of 4096 (chunks of DESC4_CHUNK tiles per thread, incremental searches as
// k4_desc).
template <int KT>
__global__ void __launch_bounds__(256) k_pull_desc(PullSrc<KT> S, uint32_t ntiles, TileDesc4* __restrict__ tiles) {
  const uint32_t nchunks = (ntiles + DESC4_CHUNK - 1) / DESC4_CHUNK;
  for (uint32_t ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks; ch += gridDim.x * blockDim.x) {
    InnerCR<KT> L, R;
    L.init(S.kp[0], S.n[0], S.kp[1], S.n[1]);
    R.init(S.kp[2], S.n[2], S.kp[3], S.n[3]);
    uint32_t aprev = 0, dprev = 0, aprev2 = 0, dprev2 = 0;
    for (uint32_t q = 0; q < DESC4_CHUNK; ++q) {
      const uint32_t tau = ch * DESC4_CHUNK + q;
      if (tau >= ntiles) break;
      const uint32_t d = tau == 0 ? 0u : (S.base / 4096u + tau) * 4096u - S.base;
      uint32_t c[4];
      const uint32_t hint = (q > 0 && d > dprev && dprev > dprev2)
                                ? aprev + (uint32_t)(((uint64_t)(aprev - aprev2) * (d - dprev)) / (dprev - dprev2))
                                : 0xFFFFFFFFu;  // as k4_desc
      const uint32_t av = corank4<KT>(L, R, d, aprev, aprev + (d - dprev), c, hint);
      aprev2 = aprev;
      dprev2 = dprev;
      aprev = av;
      dprev = d;
      TileDesc4 D;
      D.x = 0;
      D.rank = d;
      D.c[0] = c[0]; D.c[1] = c[1]; D.c[2] = c[2]; D.c[3] = c[3];
      tiles[tau] = D;
    }
  }
}

template <int KT, bool HV>
__device__ __forceinline__ void pull_issue(const TileDesc4& d, const TileDesc4* dn_or_null, const PullSrc<KT>& S,
                                           uint32_t s, unsigned char* smem, uint64_t* bars, Merge4Hdr* hdr) {
  using SM = Merge4Smem<KT, HV>;
  using K = typename KeyTraits<KT>::K;
  uint32_t c1[4];
  uint32_t rank1;
  if (dn_or_null) {
#pragma unroll
    for (int i = 0; i < 4; ++i) c1[i] = dn_or_null->c[i];
    rank1 = dn_or_null->rank;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) c1[i] = S.n[i];
    rank1 = S.N;
  }
  unsigned char* st = smem + SM::HDR + s * SM::STAGE;
  Merge4Hdr h;
  uint32_t koff = 0, voff = 0, total = 0;
  uintptr_t kg[4], vg[4];
  uint32_t kbytes[4], vbytes[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t n = c1[i] - d.c[i];
    const uintptr_t ga = (uintptr_t)(S.kp[i] + d.c[i]), ga0 = ga & ~(uintptr_t)15;
    const uint32_t bk = n ? (uint32_t)(((ga + (uintptr_t)n * sizeof(K) + 15) & ~(uintptr_t)15) - ga0) : 0u;
    h.kb[i] = (koff + (uint32_t)(ga - ga0)) / sizeof(K);
    h.n[i] = n;
    kg[i] = ga0;
    kbytes[i] = bk;
    koff += bk;
    if (HV) {
      const uintptr_t va = (uintptr_t)(S.vp[i] + d.c[i]), va0 = va & ~(uintptr_t)15;
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
  h.lo = S.base + d.rank;
  h.hi = S.base + rank1;
  h.par = 0;
  {
    const uint32_t nz = (h.n[0] != 0) + (h.n[1] != 0) + (h.n[2] != 0) + (h.n[3] != 0);
    h.mode = nz == 1 ? 2u + (h.n[0] ? 0u : h.n[1] ? 1u : h.n[2] ? 2u : 3u)
                     : ((h.n[1] == 0 && h.n[3] == 0) ? 1u : 0u);
  }
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

// Same consumer side as k4_merge_level; the producer stages the four pieces'
// windows from their own addresses.  Output keys / values at [0, N).
template <int KT, bool HV, int KQ>
__global__ void __launch_bounds__(M4_THREADS, 2) k_pull_merge(PullSrc<KT> S, typename KeyTraits<KT>::K* __restrict__ ok,
                                                              uint32_t* __restrict__ ov,
                                                              const TileDesc4* __restrict__ tiles, uint32_t count) {
  using K = typename KeyTraits<KT>::K;
  using SM = Merge4Smem<KT, HV>;
  constexpr uint32_t NT = M4_NT;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 2;
  uint64_t* ready = full + 4;
  Merge4Hdr* hdr = reinterpret_cast<Merge4Hdr*>(smem + 64);
  K* IKs = reinterpret_cast<K*>(smem + SM::HDR + SM::NSTG * SM::STAGE);
  void* IX = smem + SM::HDR + SM::NSTG * SM::STAGE + SM::IK;
  uint32_t* OVs = reinterpret_cast<uint32_t*>(smem + SM::HDR + SM::NSTG * SM::STAGE + SM::IK + SM::II);
  if (blockIdx.x >= count) return;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], NT / 32);
    mbar_init(&empty[1], NT / 32);
    mbar_init(&ready[0], 32);
    mbar_init(&ready[1], 32);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= NT) {  // producer warp
    const uint32_t plane = tid - NT;
    uint32_t it = 0;
    for (uint32_t tau = blockIdx.x; tau < count; tau += gridDim.x, ++it) {
      const uint32_t s = it % SM::NSTG;
      if (plane == 0) {
        if (it >= SM::NSTG) mbar_wait_backoff(&empty[s], ((it / SM::NSTG) - 1) & 1u);
        const TileDesc4 d = tiles[tau];
        TileDesc4 dn;
        const bool more = tau + 1 < count && (dn = tiles[tau + 1], true);
        pull_issue<KT, HV>(d, more ? &dn : nullptr, S, s, smem, full, hdr);
      }
      mbar_wait_backoff(&full[s], (it / SM::NSTG) & 1u);
      merge4_bnds<KT>(reinterpret_cast<const K*>(smem + SM::HDR + s * SM::STAGE), hdr + s, plane);
      mbar_arrive(&ready[s]);
    }
    return;
  }
  uint32_t it = 0;
  for (uint32_t tau = blockIdx.x; tau < count; tau += gridDim.x, ++it) {
    const uint32_t s = it % SM::NSTG;
    mbar_wait(&ready[s], (it / SM::NSTG) & 1u);
    merge4_tile<KT, HV>(hdr + s, smem + SM::HDR + s * SM::STAGE, IKs, IX, OVs, &empty[s], true, ok, ov, ok, ov);
  }
  if (tid == 0) bulk_wait0();
}

}  // namespace vmps
