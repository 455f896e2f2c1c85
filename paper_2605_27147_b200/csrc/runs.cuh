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

// K1+K2: descent bitmap (warp ballots) and the tile's transfer table.
template <int KT>
__global__ void __launch_bounds__(128) k_runs_tables(const typename KeyTraits<KT>::K* __restrict__ keys,
                                                     uint32_t n, uint32_t minrun, uint32_t ns,
                                                     uint32_t* __restrict__ bits_out,
                                                     uint32_t* __restrict__ tab) {
  using T = KeyTraits<KT>;
  __shared__ uint32_t sb[RT_WORDS + 2];
  __shared__ uint32_t wres[MAX_MINRUN + 2];
  const uint32_t tile = blockIdx.x;
  const uint32_t T0 = tile * RT;
  const uint32_t L = min((uint32_t)RT, n - T0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int w = warp; w <= RT_WORDS; w += 4) {
    uint32_t p = T0 + (uint32_t)w * 32u + (uint32_t)lane;
    bool b = false;
    if (p >= 1 && p < n) b = T::ord(keys[p]) < T::ord(keys[p - 1]);
    uint32_t word = __ballot_sync(0xFFFFFFFFu, b);
    if (lane == 0) {
      sb[w] = word;
      if (w < RT_WORDS && T0 + (uint32_t)w * 32u < n) bits_out[tile * RT_WORDS + w] = word;
    }
  }
  if (threadIdx.x == 0) sb[RT_WORDS + 1] = 0;
  __syncthreads();
  TileCtx c{sb, T0, L, n, minrun};
  // walks from START(o) (o < minrun) and from the first set / clear bit
  uint32_t d_asc = find_bit(sb, 0, L, true);
  uint32_t d_desc = find_bit(sb, 0, L, false);
  for (uint32_t w = threadIdx.x; w < minrun + 2; w += blockDim.x) {
    uint32_t x = w < minrun ? w : (w == minrun ? d_asc : d_desc);
    uint32_t res;
    if (x >= L || T0 + x >= n) {
      res = ST_END << 24;  // unused / not reachable
    } else {
      uint32_t cnt = 0;
      uint32_t st = tile_walk<false>(c, x, &cnt, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
      res = (st << 24) | cnt;
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
                            uint64_t* __restrict__ entry) {
  if (threadIdx.x != 0) return;
  uint32_t st = 0, cnt = 0;
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

// K4: re-walk each tile from its entry state and emit run starts and kinds.
__global__ void __launch_bounds__(32) k_runs_emit(const uint32_t* __restrict__ gbits, uint32_t n,
                                                  uint32_t minrun,
                                                  const uint64_t* __restrict__ entry,
                                                  uint32_t* __restrict__ run_start,
                                                  uint8_t* __restrict__ run_kind,
                                                  uint32_t* __restrict__ scalars) {
  __shared__ uint32_t sb[RT_WORDS + 2];
  const uint32_t tile = blockIdx.x;
  const uint32_t T0 = tile * RT;
  const uint32_t L = min((uint32_t)RT, n - T0);
  const uint32_t nwords = (n + 31) / 32;
  for (uint32_t w = threadIdx.x; w < RT_WORDS + 2; w += blockDim.x) {
    uint32_t gw = tile * RT_WORDS + w;
    sb[w] = gw < nwords ? gbits[gw] : 0u;
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  TileCtx c{sb, T0, L, n, minrun};
  uint64_t e = entry[tile];
  uint32_t st = (uint32_t)(e >> 32), idx = (uint32_t)e;
  uint32_t d_asc = find_bit(sb, 0, L, true);
  uint32_t d_desc = find_bit(sb, 0, L, false);
  uint32_t x, out, rev_open;
  uint32_t n_rev = 0, n_ext = 0;
  bool ended = false;
  if (resolve_entry(c, st, d_asc, d_desc, &x, &out, &rev_open)) {
    n_rev += rev_open;
    uint32_t cnt = 0;
    out = tile_walk<true>(c, x, &cnt, run_start, run_kind, gbits, &idx, &n_rev, &n_ext);
    ended = out == ST_END;
  } else {
    n_rev += rev_open;
    ended = (st != ST_END) && out == ST_END;
  }
  if (n_rev) atomicAdd(&scalars[SC_REVERSED], n_rev);
  if (n_ext) atomicAdd(&scalars[SC_EXTENDED], n_ext);
  if (ended) {
    scalars[SC_RUNS] = idx;
    run_start[idx] = n;  // sentinel s_r = n
  }
}

}  // namespace vmps
