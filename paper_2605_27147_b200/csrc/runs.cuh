// runs.cuh -- run detection (ExtractRun, P:399 / P:756, reading R3)
// as a data-parallel chain over tiles.
//
// bit p = key[p] < key[p-1] (a descent).  A run starting at s is strictly
// descending iff bit[s+1] (it then ends at the first clear bit at >= s+2),
// else ascending (it ends at the first set bit at >= s+1); its end is
// min(n, max(natural end, s + minrun)).  The run starts form a chain
// s -> end(s).  At each tile boundary B the chain is in one state:
//   START(o)  the next run starts at B + o           (o < minrun)
//   ASC(f)    an ascending run is open at B; it ends at
//             max(first set bit >= B, B + f)          (f < minrun)
//   DESC(f)   a descending run is open at B; it ends at
//             max(first clear bit >= B, B + f)
//   END       the chain reached n
// Each tile computes its transfer table state -> (state at its right end,
// runs started inside it); tables compose associatively (a scan over tiles),
// and a re-walk from each tile's entry state emits run starts and kinds.
#pragma once
#include "vmps_internal.cuh"

namespace vmps {

__device__ __forceinline__ uint32_t st_start(uint32_t o) { return o; }
__device__ __forceinline__ uint32_t st_asc(uint32_t f, uint32_t mr) { return mr + f; }
__device__ __forceinline__ uint32_t st_desc(uint32_t f, uint32_t mr) { return 2 * mr + f; }

// first position q in [rel, lim) whose bit equals want (positions relative to
// the bitmap base `sb`); lim if none.
__device__ __forceinline__ uint32_t find_bit(const uint32_t* sb, uint32_t rel, uint32_t lim,
                                             bool want) {
  while (rel < lim) {
    uint32_t w = sb[rel >> 5];
    if (!want) w = ~w;
    w &= (~0u) << (rel & 31u);
    if (w) {
      uint32_t q = (rel & ~31u) + (uint32_t)(__ffs(w) - 1);
      return q < lim ? q : lim;
    }
    rel = (rel & ~31u) + 32u;
  }
  return lim;
}

__device__ __forceinline__ bool get_bit(const uint32_t* sb, uint32_t rel) {
  return (sb[rel >> 5] >> (rel & 31u)) & 1u;
}

struct TileCtx {
  const uint32_t* sb;  // bits of positions [T0, T0 + L + 1] (relative)
  uint32_t T0, L, n, minrun;
};

// Walk the chain from run start x (relative, x < L, T0 + x < n) to the tile's
// right end.  If EMIT, write run starts/kinds from index *idx on.
template <bool EMIT>
__device__ uint32_t tile_walk(const TileCtx& c, uint32_t x, uint32_t* cnt, uint32_t* run_start,
                              uint8_t* run_kind, const uint32_t* gbits, uint32_t* idx,
                              uint32_t* n_rev, uint32_t* n_ext) {
  for (;;) {
    uint32_t gx = c.T0 + x;
    (*cnt)++;
    bool last = gx + 1 >= c.n;
    bool desc = !last && get_bit(c.sb, x + 1);  // x + 1 <= L: peek allowed
    if (EMIT) {
      // kind: EXT iff the natural end lies before gx + minrun (or n - gx < minrun)
      uint32_t wlim = min(c.n, gx + c.minrun);
      bool ext;
      if (gx + c.minrun > c.n) {
        ext = true;
      } else {
        uint32_t from = desc ? gx + 2 : gx + 1;
        ext = from < wlim && find_bit(gbits, from, wlim, !desc) < wlim;
      }
      run_start[*idx] = gx;
      run_kind[*idx] = (uint8_t)((desc ? VMPS_RUN_DESC : 0u) | (ext ? VMPS_RUN_EXT : 0u));
      (*idx)++;
      if (ext) (*n_ext)++;
    }
    if (last) return ST_END;
    uint32_t nat = desc ? find_bit(c.sb, x + 2, c.L, false) : find_bit(c.sb, x + 1, c.L, true);
    if (nat >= c.L) {  // the run is open at the tile's right end
      if (c.T0 + c.L >= c.n) {
        if (EMIT && desc) *n_rev += c.n - gx;
        return ST_END;
      }
      if (EMIT && desc) *n_rev += c.T0 + c.L - gx;  // rest counted by the next tile
      uint32_t f = (x + c.minrun > c.L) ? x + c.minrun - c.L : 0u;
      return desc ? st_desc(f, c.minrun) : st_asc(f, c.minrun);
    }
    if (EMIT && desc) *n_rev += nat - x;
    uint32_t e = max(nat, x + c.minrun);
    if (c.T0 + e >= c.n) return ST_END;
    if (e >= c.L) return st_start(e - c.L);
    x = e;
  }
}

// Resolve an entry state of this tile: returns the first run start inside
// the tile (relative) or writes the out-state directly.
// Returns true and sets *x when a run starts inside the tile.
__device__ __forceinline__ bool resolve_entry(const TileCtx& c, uint32_t s, uint32_t d_asc,
                                              uint32_t d_desc, uint32_t* x, uint32_t* out,
                                              uint32_t* rev_open) {
  uint32_t mr = c.minrun;
  *rev_open = 0;
  if (s == ST_END) { *out = ST_END; return false; }
  uint32_t e;
  if (s < mr) {
    e = s;
  } else {
    bool desc = s >= 2 * mr;
    uint32_t f = desc ? s - 2 * mr : s - mr;
    uint32_t d = desc ? d_desc : d_asc;
    if (d >= c.L) {  // still open across the whole tile
      if (desc) *rev_open = c.L;
      if (c.T0 + c.L >= c.n) { *out = ST_END; return false; }
      uint32_t nf = f > c.L ? f - c.L : 0u;
      *out = desc ? st_desc(nf, mr) : st_asc(nf, mr);
      return false;
    }
    if (desc) *rev_open = d;
    e = max(d, f);
  }
  if (c.T0 + e >= c.n) { *out = ST_END; return false; }
  if (e >= c.L) { *out = st_start(e - c.L); return false; }
  *x = e;
  return true;
}

// Per-word suffix tables of a tile: fs[w] / fc[w] = first position >= 32w in
// [0, L) whose bit is set / clear (L if none).  One warp.
__device__ __forceinline__ void tile_suffix_tables(const uint32_t* sb, uint32_t L, uint16_t* fs, uint16_t* fc,
                                                   int lane) {
  // each lane owns words [5 lane, 5 lane + 5) (covers 160 >= RT_WORDS + 1 words)
  constexpr int PER = 5;
  uint32_t ls = L, lc = L;  // first set / clear within the lane's words
  uint32_t vs[PER], vc[PER];
#pragma unroll
  for (int q = PER - 1; q >= 0; --q) {
    const uint32_t w = (uint32_t)lane * PER + q;
    uint32_t setm = 0, clrm = 0;
    if (32 * w < L) {
      const uint32_t nvalid = min(32u, L - 32 * w);
      const uint32_t vm = nvalid == 32 ? 0xFFFFFFFFu : ((1u << nvalid) - 1u);
      setm = sb[w] & vm;
      clrm = ~sb[w] & vm;
    }
    if (setm) ls = 32 * w + (uint32_t)(__ffs(setm) - 1);
    if (clrm) lc = 32 * w + (uint32_t)(__ffs(clrm) - 1);
    vs[q] = ls;
    vc[q] = lc;
  }
  // suffix-min across lanes: the first hit of all later lanes
  uint32_t ns = ls, nc = lc;  // lane's own first (= value at its first word)
  uint32_t as = L, ac = L;    // min over lanes > me
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t ys = __shfl_down_sync(0xFFFFFFFFu, ns, o);
    const uint32_t yc = __shfl_down_sync(0xFFFFFFFFu, nc, o);
    if (lane + o < 32) { ns = min(ns, ys); nc = min(nc, yc); }
  }
  as = __shfl_down_sync(0xFFFFFFFFu, ns, 1);
  ac = __shfl_down_sync(0xFFFFFFFFu, nc, 1);
  if (lane == 31) { as = L; ac = L; }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const uint32_t w = (uint32_t)lane * PER + q;
    if (w <= RT_WORDS + 1) {
      fs[w] = (uint16_t)min(vs[q], as);
      fc[w] = (uint16_t)min(vc[q], ac);
    }
  }
}

// first set (want) / clear bit at position >= p within [0, L), via the tables
__device__ __forceinline__ uint32_t tile_first(const uint32_t* sb, const uint16_t* ft, uint32_t p, uint32_t L,
                                               bool want) {
  if (p >= L) return L;
  const uint32_t w = p >> 5;
  uint32_t m = want ? sb[w] : ~sb[w];
  m &= (~0u) << (p & 31u);
  if (32 * w + 32 > L) m &= (L - 32 * w >= 32) ? 0xFFFFFFFFu : ((1u << (L - 32 * w)) - 1u);
  if (m) return 32 * w + (uint32_t)(__ffs(m) - 1);
  return ft[w + 1];
}

// The tile's descent bits: thread t builds word t (positions T0+32t ..
// T0+32t+31) from its keys and the key before them; the peek bit at T0+RT
// (first bit of word RT_WORDS) comes from thread 0.  128-bit loads when the
// whole word lies inside [0, n).
template <int KT>
__device__ __forceinline__ void build_tile_bits(const typename KeyTraits<KT>::K* __restrict__ keys, uint32_t n,
                                                uint32_t T0, uint32_t* sb, uint32_t* __restrict__ gout,
                                                const typename KeyTraits<KT>::K* __restrict__ prev,
                                                const typename KeyTraits<KT>::K* __restrict__ halo,
                                                uint32_t n_halo) {
  // keys[0, n) is the array (or a shard of it); positions n .. n + n_halo - 1
  // are the next shards' first keys (halo) and *prev the previous shard's last
  // key (bit 0 = the descent into this shard), so a shard's bitmap is the
  // global one
  using T = KeyTraits<KT>;
  using K = typename T::K;
  auto key = [&](uint32_t p) -> K { return p < n ? keys[p] : halo[p - n]; };
  const uint32_t nx = n + n_halo;
  const uint32_t t = threadIdx.x;  // blockDim.x == RT_WORDS
  const uint32_t p0 = T0 + 32u * t;
  uint32_t word = 0;
  if (p0 + 32 <= n && p0 >= 1) {
    K k[32];
    const uint4* src = reinterpret_cast<const uint4*>(keys + p0);
    constexpr int PER = 16 / sizeof(K);
#pragma unroll
    for (int q = 0; q < 32 / PER; ++q) {
      uint4 v = __ldg(src + q);
      const K* e = reinterpret_cast<const K*>(&v);
#pragma unroll
      for (int r = 0; r < PER; ++r) k[q * PER + r] = e[r];
    }
    word = T::ord(k[0]) < T::ord(keys[p0 - 1]) ? 1u : 0u;
#pragma unroll
    for (int l = 1; l < 32; ++l) word |= (T::ord(k[l]) < T::ord(k[l - 1]) ? 1u : 0u) << l;
  } else {
    for (uint32_t l = 0; l < 32; ++l) {
      const uint32_t p = p0 + l;
      if (p == 0) word |= (prev && T::ord(keys[0]) < T::ord(*prev)) ? 1u : 0u;
      else if (p < nx && T::ord(key(p)) < T::ord(key(p - 1))) word |= 1u << l;
    }
  }
  sb[t] = word;
  if (p0 < nx) gout[t] = word;
  if (T0 + RT >= n && t < 8) {  // last tile of a shard: the halo's words past the tile
    const uint32_t q0 = T0 + RT + 32u * t;
    if (q0 < nx) {
      uint32_t hw = 0;
      for (uint32_t l = 0; l < 32; ++l) {
        const uint32_t p = q0 + l;
        if (p < nx && T::ord(key(p)) < T::ord(key(p - 1))) hw |= 1u << l;
      }
      gout[RT_WORDS + t] = hw;
    }
  }
  if (t == 0) {
    const uint32_t p = T0 + RT;
    sb[RT_WORDS] = (p < nx && T::ord(key(p)) < T::ord(key(p - 1))) ? 1u : 0u;
    sb[RT_WORDS + 1] = 0;
  }
}

// Long-run masks of one bitmap word (thread-per-word).  For a run start x
// with x + m < L the run is "short" iff its natural end is <= x + m (the run
// then ends at x + m, ExtractRun's minrun extension) and "long"
// otherwise (it ends at its natural end > x + m):
//   la bit x: ascending run from x is long  <=> no descent in [x+1, x+m]
//   ld bit x: descending run from x is long <=> descents at all of [x+1, x+m]
// Sliding-window AND of width m (1 <= m <= 64) over the 96 bits of words
// w, w+1, w+2 by doubling; bits past the tile are never consulted because
// every window used lies inside [1, L-1].
__device__ __forceinline__ uint32_t window_and_m(unsigned __int128 b, uint32_t m) {
  uint32_t p = 1;  // b bit i: AND of [i, i+p)
  while (2 * p <= m) {
    b &= b >> p;
    p *= 2;
  }
  b &= b >> (m - p);         // m - p < p: two overlapping windows cover [i, i+m)
  return (uint32_t)(b >> 1);  // bit i: AND of [i+1, i+m]
}
// m <= 32 (minrun 32 for every n = 2^k): the windows [i+1, i+m] of the
// word's 32 starts end at bit 63 at most, so 64-bit arithmetic suffices.
__device__ __forceinline__ uint32_t window_and_m64(uint64_t b, uint32_t m) {
  uint32_t p = 1;
  while (2 * p <= m) {
    b &= b >> p;
    p *= 2;
  }
  b &= b >> (m - p);
  return (uint32_t)(b >> 1);
}
__device__ __forceinline__ void long_masks(const uint32_t* sb, uint32_t w, uint32_t m, uint32_t* la,
                                           uint32_t* ld) {
  if (m <= 32) {
    const uint64_t b = (uint64_t)sb[w] | ((uint64_t)sb[w + 1] << 32);
    ld[w] = window_and_m64(b, m);
    la[w] = window_and_m64(~b, m);
    return;
  }
  const unsigned __int128 b = (unsigned __int128)sb[w] | ((unsigned __int128)sb[w + 1] << 32) |
                              ((unsigned __int128)sb[w + 2] << 64);
  const unsigned __int128 nb = ~b & (((unsigned __int128)1 << 96) - 1);
  ld[w] = window_and_m(b, m);
  la[w] = window_and_m(nb, m);
}

// minrun == 32 (every n = 2^k >= 64): a short run at x = 32 w + b hands over
// to 32 (w + 1) + b, the same bit of the next bitmap word.  stop[b] is a
// 128-bit mask over the tile's words of the positions 32 w + b where that
// stops (a long run, or a run reaching the tile's end: x + 32 >= L), built
// by warp ballots (a transpose of the per-word stop masks), so a walker skips
// a whole stretch of short runs with one find-first-set.
__device__ __forceinline__ void stop_masks32(const uint32_t* sb, const uint32_t* la, const uint32_t* ld, uint32_t L,
                                             uint32_t* ts) {
  const uint32_t w = threadIdx.x, lane = w & 31u, k = w >> 5;  // one thread per word
  const uint32_t dw = (sb[w] >> 1) | (sb[w + 1] << 31);        // bit b: descent at 32 w + b + 1
  uint32_t st = (dw & ld[w]) | (~dw & la[w]);
  const int lim = (int)L - 32 - (int)(32 * w);                  // bits b >= lim have x + 32 >= L
  if (lim <= 0) st = 0xFFFFFFFFu;
  else if (lim < 32) st |= 0xFFFFFFFFu << lim;
  // 32x32 bit transpose across the warp (lane l's bit b -> lane b's bit l):
  // five butterfly exchanges instead of 32 ballots
  uint32_t x = st;
#pragma unroll
  for (uint32_t j = 16; j >= 1; j >>= 1) {
    const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                     : j == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y << j) & ~m));
  }
  ts[4 * lane + k] = x;
}
// first word >= w whose bit b is a stop (128 if none)
__device__ __forceinline__ uint32_t next_stop32(const uint32_t* ts, uint32_t b, uint32_t w) {
  for (uint32_t k = w >> 5; k < 4; ++k) {
    uint32_t v = ts[4 * b + k];
    if (k == (w >> 5)) v &= 0xFFFFFFFFu << (w & 31u);
    if (v) return 32 * k + (uint32_t)(__ffs(v) - 1);
  }
  return 128;
}

// Walk the chain from in-tile run start x (T0 + x < n) until it leaves the
// tile; returns the exit state, counts the starts visited and, if MARK, sets
// them in `startb`.  ExtractRun, P:399 / P:756, reading R3.
// With ts (minrun == 32) stretches of short runs are skipped in O(1).
template <bool MARK>
__device__ __forceinline__ uint32_t tile_walk_fast(const uint32_t* sb, const uint32_t* la, const uint32_t* ld,
                                                   const uint16_t* fs, const uint16_t* fc, uint32_t T0,
                                                   uint32_t L, uint32_t n, uint32_t m, uint32_t x,
                                                   uint32_t* cnt, uint32_t* startb, const uint32_t* ts = nullptr) {
  const bool last_tile = T0 + L >= n;
  uint32_t c = 0;
  uint32_t out;
  for (;;) {
    if (ts) {  // skip the short runs at bit b up to the next stop
      const uint32_t b = x & 31u, w = x >> 5;
      const uint32_t w2 = next_stop32(ts, b, w);
      if (w2 > w && w2 < 128) {
        c += w2 - w;
        if (MARK)
          for (uint32_t ww = w; ww < w2; ++ww) startb[ww] |= 1u << b;
        x = 32 * w2 + b;
      }
    }
    ++c;
    if (MARK) startb[x >> 5] |= 1u << (x & 31u);
    if (T0 + x + 1 >= n) { out = ST_END; break; }
    const bool desc = get_bit(sb, x + 1);  // x + 1 <= L: peek allowed
    if (x + m < L) {
      if (!get_bit(desc ? ld : la, x)) { x += m; continue; }  // short run: ends at x + m
      const uint32_t nat = tile_first(sb, desc ? fc : fs, x + m + 1, L, !desc);
      if (nat >= L) { out = last_tile ? ST_END : (desc ? st_desc(0u, m) : st_asc(0u, m)); break; }
      x = nat;
      continue;
    }
    // the run reaches the tile's right end
    const uint32_t nat = desc ? tile_first(sb, fc, x + 2, L, false) : tile_first(sb, fs, x + 1, L, true);
    if (nat >= L) { out = last_tile ? ST_END : (desc ? st_desc(x + m - L, m) : st_asc(x + m - L, m)); break; }
    out = (T0 + x + m >= n) ? ST_END : st_start(x + m - L);
    break;
  }
  *cnt = c;
  return out;
}

// K1+K2: descent bitmap, long-run masks and the tile's transfer table: one
// walker per entry class (offsets 0..m-1, open ascending, open descending).
// n: keys in this array / shard; n_end: the position where the chain ends
// (= n for a whole array or the last shard, 0xFFFFFFFF for an inner shard);
// prev / halo: see build_tile_bits.
template <int KT>
__global__ void __launch_bounds__(128) k_runs_tables(const typename KeyTraits<KT>::K* __restrict__ keys,
                                                     uint32_t n, uint32_t minrun, uint32_t ns,
                                                     uint32_t* __restrict__ bits_out,
                                                     uint32_t* __restrict__ tab, uint32_t n_end,
                                                     const typename KeyTraits<KT>::K* __restrict__ prev,
                                                     const typename KeyTraits<KT>::K* __restrict__ halo,
                                                     uint32_t n_halo) {
  __shared__ uint32_t sb[RT_WORDS + 2];
  __shared__ uint32_t la[RT_WORDS], ld[RT_WORDS];
  __shared__ uint16_t fs[RT_WORDS + 2], fc[RT_WORDS + 2];
  __shared__ uint32_t wres[MAX_MINRUN + 2];
  __shared__ uint32_t ts[32 * 4];
  static_assert(RT_WORDS == 128, "one thread per bitmap word");
  const uint32_t tile = blockIdx.x;
  const uint32_t T0 = tile * RT;
  const uint32_t L = min((uint32_t)RT, n - T0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  build_tile_bits<KT>(keys, n, T0, sb, bits_out + (size_t)tile * RT_WORDS, prev, halo, n_halo);
  if (threadIdx.x == 0) sb[RT_WORDS + 1] = 0;
  __syncthreads();
  if (warp == 0) tile_suffix_tables(sb, L, fs, fc, lane);
  long_masks(sb, threadIdx.x, minrun, la, ld);
  __syncthreads();
  const bool m32 = minrun == 32;
  if (m32) {
    stop_masks32(sb, la, ld, L, ts);
    __syncthreads();
  }
  const uint32_t d_asc = fs[0], d_desc = fc[0];
  TileCtx c{sb, T0, L, n_end, minrun};
  for (uint32_t w = threadIdx.x; w < minrun + 2; w += blockDim.x) {
    uint32_t x = w < minrun ? w : (w == minrun ? d_asc : d_desc);
    uint32_t res;
    if (x >= L || T0 + x >= n) {
      res = ST_END << 24;  // unused / not reachable
    } else {
      uint32_t cnt = 0;
      const uint32_t v = tile_walk_fast<false>(sb, la, ld, fs, fc, T0, L, n_end, minrun, x, &cnt, nullptr,
                                               m32 ? ts : nullptr);
      res = (v << 24) | cnt;
    }
    wres[w] = res;
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < ns; s += blockDim.x) {
    uint32_t x, out, rev;
    uint32_t v;
    if (resolve_entry(c, s, d_asc, d_desc, &x, &out, &rev)) {
      // x < minrun: the walk from offset x.  Otherwise x = max(d, f) = d with
      // d the first set (ASC) / clear (DESC) bit, since f < minrun.
      if (x < minrun) v = wres[x];
      else v = (s >= 2 * minrun) ? wres[minrun + 1] : wres[minrun];
    } else {
      v = out << 24;
    }
    tab[(size_t)tile * ns + s] = v;
  }
}

// Compose groups of CHAIN_G consecutive tables (level l -> l+1).
template <typename In>
__device__ __forceinline__ void unpack(In v, uint32_t* st, uint32_t* cnt);
template <>
__device__ __forceinline__ void unpack<uint32_t>(uint32_t v, uint32_t* st, uint32_t* cnt) {
  *st = v >> 24;
  *cnt = v & 0xFFFFFFu;
}
template <>
__device__ __forceinline__ void unpack<uint64_t>(uint64_t v, uint32_t* st, uint32_t* cnt) {
  *st = (uint32_t)(v >> 32);
  *cnt = (uint32_t)v;
}

template <typename In>
__global__ void __launch_bounds__(256) k_chain_compose(const In* __restrict__ in, uint32_t m,
                                                       uint32_t ns, uint64_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  In* s = reinterpret_cast<In*>(smem_raw);
  const uint32_t g0 = blockIdx.x * CHAIN_G;
  const uint32_t gm = min((uint32_t)CHAIN_G, m - g0);
  for (uint32_t q = threadIdx.x; q < gm * ns; q += blockDim.x) s[q] = in[(size_t)g0 * ns + q];
  __syncthreads();
  for (uint32_t st0 = threadIdx.x; st0 < ns; st0 += blockDim.x) {
    uint32_t st = st0, cnt = 0;
    for (uint32_t t = 0; t < gm && st != ST_END; ++t) {
      uint32_t s2, c2;
      unpack<In>(s[t * ns + st], &s2, &c2);
      st = s2;
      cnt += c2;
    }
    out[(size_t)blockIdx.x * ns + st0] = ((uint64_t)st << 32) | cnt;
  }
}

// Sequential walk over <= CHAIN_G tables of the top level from START(0).
template <typename In>
__global__ void k_chain_top(const In* __restrict__ in, uint32_t m, uint32_t ns,
                            uint64_t* __restrict__ entry, uint32_t st0) {
  if (threadIdx.x != 0) return;
  uint32_t st = st0, cnt = 0;
  for (uint32_t t = 0; t < m; ++t) {
    entry[t] = ((uint64_t)st << 32) | cnt;
    if (st != ST_END) {
      uint32_t s2, c2;
      unpack<In>(in[(size_t)t * ns + st], &s2, &c2);
      st = s2;
      cnt += c2;
    }
  }
}

// A shard's transfer table: for every entry state, walk the <= CHAIN_G tables
// of the top level (one thread per state): (exit state << 32) | runs started.
template <typename In>
__global__ void k_chain_all(const In* __restrict__ in, uint32_t m, uint32_t ns, uint64_t* __restrict__ out) {
  for (uint32_t s0 = threadIdx.x; s0 < ns; s0 += blockDim.x) {
    uint32_t st = s0, cnt = 0;
    for (uint32_t t = 0; t < m && st != ST_END; ++t) {
      uint32_t s2, c2;
      unpack<In>(in[(size_t)t * ns + st], &s2, &c2);
      st = s2;
      cnt += c2;
    }
    out[s0] = ((uint64_t)st << 32) | cnt;
  }
}

// Expand entries of level l+1 groups to their CHAIN_G members at level l.
template <typename In>
__global__ void __launch_bounds__(256) k_chain_expand(const In* __restrict__ in, uint32_t m,
                                                      uint32_t ns, const uint64_t* __restrict__ gentry,
                                                      uint64_t* __restrict__ entry) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  In* s = reinterpret_cast<In*>(smem_raw);
  const uint32_t g0 = blockIdx.x * CHAIN_G;
  const uint32_t gm = min((uint32_t)CHAIN_G, m - g0);
  for (uint32_t q = threadIdx.x; q < gm * ns; q += blockDim.x) s[q] = in[(size_t)g0 * ns + q];
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t e = gentry[blockIdx.x];
  uint32_t st = (uint32_t)(e >> 32), cnt = (uint32_t)e;
  for (uint32_t t = 0; t < gm; ++t) {
    entry[g0 + t] = ((uint64_t)st << 32) | cnt;
    if (st != ST_END) {
      uint32_t s2, c2;
      unpack<In>(s[t * ns + st], &s2, &c2);
      st = s2;
      cnt += c2;
    }
  }
}

// K4: re-walk each tile from its entry state (pointer chasing over nxt),
// mark the run starts, then emit starts and kinds in parallel.
__global__ void __launch_bounds__(128) k_runs_emit(const uint32_t* __restrict__ gbits, uint32_t n,
                                                   uint32_t minrun,
                                                   const uint64_t* __restrict__ entry,
                                                   uint32_t* __restrict__ run_start,
                                                   uint8_t* __restrict__ run_kind,
                                                   uint32_t* __restrict__ scalars, uint32_t n_end,
                                                   uint32_t n_halo) {
  __shared__ uint32_t sb[RT_WORDS + 4];
  __shared__ uint16_t fs[RT_WORDS + 2], fc[RT_WORDS + 2];
  __shared__ uint32_t startb[RT_WORDS];
  __shared__ uint32_t la[RT_WORDS], ld[RT_WORDS];
  __shared__ uint32_t ts[32 * 4];
  __shared__ uint32_t wsum[4];
  __shared__ uint32_t s_idx0, s_rev;
  const uint32_t tile = blockIdx.x;
  const uint32_t T0 = tile * RT;
  const uint32_t L = min((uint32_t)RT, n - T0);
  const uint32_t nwords = (n + n_halo + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t w = threadIdx.x; w < RT_WORDS + 4; w += blockDim.x) {
    const uint32_t gw = tile * RT_WORDS + w;
    sb[w] = gw < nwords ? gbits[gw] : 0u;
  }
  if (threadIdx.x < RT_WORDS) startb[threadIdx.x] = 0u;
  __syncthreads();
  if (warp == 0) tile_suffix_tables(sb, L, fs, fc, lane);
  long_masks(sb, threadIdx.x, minrun, la, ld);
  __syncthreads();
  const bool m32 = minrun == 32;
  if (m32) {
    stop_masks32(sb, la, ld, L, ts);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    TileCtx c{sb, T0, L, n_end, minrun};
    const uint64_t e = entry[tile];
    const uint32_t st = (uint32_t)(e >> 32);
    uint32_t x, out, rev_open, cnt = 0;
    bool ended;
    if (resolve_entry(c, st, fs[0], fc[0], &x, &out, &rev_open)) {
      ended = tile_walk_fast<true>(sb, la, ld, fs, fc, T0, L, n_end, minrun, x, &cnt, startb, m32 ? ts : nullptr) ==
              ST_END;
    } else {
      ended = (st != ST_END) && out == ST_END;
    }
    s_idx0 = (uint32_t)e;
    s_rev = rev_open;
    if (ended) {
      scalars[SC_RUNS] = (uint32_t)e + cnt;
      run_start[(uint32_t)e + cnt] = n;  // sentinel s_r = n
    }
  }
  __syncthreads();
  // exclusive scan of the per-word start counts (thread t = word t)
  const uint32_t t = threadIdx.x;
  const uint32_t bits = startb[t];
  const uint32_t c = (uint32_t)__popc(bits);
  uint32_t incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  uint32_t off = incl - c;
  for (int q = 0; q < warp; ++q) off += wsum[q];
  uint32_t idx = s_idx0 + off;
  uint32_t n_rev = 0, n_ext = 0;
  for (uint32_t m = bits; m; m &= m - 1) {
    const uint32_t x = 32 * t + (uint32_t)(__ffs(m) - 1);
    const uint32_t gx = T0 + x;
    const bool last = gx + 1 >= n_end;
    const bool desc = !last && get_bit(sb, x + 1);
    bool ext;
    if (gx + minrun > n_end) {
      ext = true;
    } else {  // a breaking bit inside [from, x + minrun) (at most 64 bits past the tile)
      const uint32_t from = desc ? x + 2 : x + 1;
      const uint32_t lim = x + minrun;
      ext = from < lim && find_bit(sb, from, lim, !desc) < lim;
    }
    if (desc) {
      const uint32_t nat = tile_first(sb, fc, x + 2, L, false);
      n_rev += (nat < L ? nat : L) - x;  // the part in later tiles is counted there
    }
    run_start[idx] = gx;
    run_kind[idx] = (uint8_t)((desc ? VMPS_RUN_DESC : 0u) | (ext ? VMPS_RUN_EXT : 0u));
    ++idx;
    if (ext) ++n_ext;
  }
  if (t == 0) n_rev += s_rev;
  for (int o = 16; o; o >>= 1) {
    n_rev += __shfl_xor_sync(0xFFFFFFFFu, n_rev, o);
    n_ext += __shfl_xor_sync(0xFFFFFFFFu, n_ext, o);
  }
  if (lane == 0) {
    if (n_rev) atomicAdd(&scalars[SC_REVERSED], n_rev);
    if (n_ext) atomicAdd(&scalars[SC_EXTENDED], n_ext);
  }
}

}  // namespace vmps
