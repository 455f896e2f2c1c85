// leaf_radix.cuh -- leaf engine, radix form.
//
// A leaf batch is a run of consecutive touching units (maximal subtrees of
// the merge tree with <= Z elements); each unit's
// output is the stable sort of its segment under the key order (a stable
// sort's output is unique, so it equals merging the unit's runs along the
// Powersort tree, with ties to the left run).
//
// The batch (<= LEAF_CAP elements) is sorted in shared memory by an LSD radix
// sort of the key order image (8-bit digits, stable passes) followed by a
// stable pass over the unit index: the result is grouped by unit, sorted by
// key within a unit, and equal keys keep their input order.  Digits whose
// bits are equal over the whole batch are skipped (OR / AND of the images),
// as is the unit pass of a single-unit batch.
//
// Layout: warp w owns positions [32 K w, 32 K (w + 1)) with K = LEAF_K items
// per lane (11 with the default 384-thread CTAs: 12 warps x 352 positions),
// striped (lane l, item i <-> position 32 K w + 32 i + l), so global
// loads / stores are coalesced and
// processing items in order (i outer, lanes inner) is position order, which
// makes the warp-level ranking (match.any + per-warp digit counters) stable.
#pragma once
#include "engine.cuh"

namespace vmps {

constexpr int LR_WARPS = LEAF_THREADS / 32;      // 12 (384 threads)
constexpr int LR_ITEMS = LEAF_K;                 // 11
constexpr int LR_SPAN = 32 * LR_ITEMS;           // 352 positions per warp
static_assert(LR_WARPS * LR_SPAN == LEAF_CAP, "leaf radix layout");

template <int KT>
struct LeafRadixSmem {
  using O = typename KeyTraits<KT>::O;
  static constexpr uint32_t NW = LEAF_CAP / 32 + 1;  // bitmap words
  static constexpr uint32_t IMG = 2 * LEAF_CAP * sizeof(O);
  static constexpr uint32_t IDX = 2 * LEAF_CAP * 2;
  static constexpr uint32_t CNT = LR_WARPS * 256 * 4;
  static constexpr uint32_t BITS = 4 * NW * 4;
  static constexpr uint32_t MISC = 64;
  static constexpr uint32_t BYTES = IMG + IDX + CNT + BITS + MISC;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <int KT, bool HV>
__global__ void __launch_bounds__(LEAF_THREADS, 2) k_leaf_radix(
    typename KeyTraits<KT>::K* __restrict__ k0, uint32_t* __restrict__ v0,
    typename KeyTraits<KT>::K* __restrict__ k1, uint32_t* __restrict__ v1,
    const uint32_t* __restrict__ units, const uint32_t* __restrict__ batch_first) {
  using T = KeyTraits<KT>;
  using K = typename T::K;
  using O = typename T::O;
  using SM = LeafRadixSmem<KT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  O* const simg = reinterpret_cast<O*>(smem_raw);                                  // 2 x LEAF_CAP
  uint16_t* const sidx = reinterpret_cast<uint16_t*>(smem_raw + SM::IMG);          // 2 x LEAF_CAP
  uint32_t* const cnt = reinterpret_cast<uint32_t*>(smem_raw + SM::IMG + SM::IDX);  // [warp][256]
  uint32_t* const ubits = cnt + LR_WARPS * 256;  // unit-start bitmap
  uint32_t* const upre = ubits + SM::NW;         // exclusive popcount prefix per word
  uint32_t* const pcar = upre + SM::NW;          // parity of the unit open at each word's end
  uint32_t* const pbits = pcar + SM::NW;         // parity bit at each unit start
  uint32_t* const misc = pbits + SM::NW;         // [0..1] OR, [2..3] AND of images; [4..11] warp sums

  const uint32_t x0 = batch_first[blockIdx.x], x1 = batch_first[blockIdx.x + 1];
  if (x0 >= x1) return;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t bstart = units[3 * x0];
  const uint32_t E = units[3 * (x1 - 1) + 1] - bstart;
  const uint32_t nunits = x1 - x0;
  const uint32_t nwords = (E + 31) / 32;
  for (uint32_t w = tid; w < nwords; w += LEAF_THREADS) { ubits[w] = 0u; pbits[w] = 0u; }
  if (tid == 0) { misc[0] = misc[1] = 0u; misc[2] = misc[3] = 0xFFFFFFFFu; }
  __syncthreads();
  for (uint32_t x = x0 + tid; x < x1; x += LEAF_THREADS) {
    const uint32_t q = units[3 * x] - bstart;
    atomicOr(&ubits[q >> 5], 1u << (q & 31u));
    if (units[3 * x + 2]) atomicOr(&pbits[q >> 5], 1u << (q & 31u));
  }

  // striped load of the order images; OR / AND find the digits that vary
  const uint32_t wbase = warp * LR_SPAN + lane;
  O img[LR_ITEMS];
  uint32_t ix[LR_ITEMS];
  O vor = 0, vand = ~O(0);
#pragma unroll
  for (int i = 0; i < LR_ITEMS; ++i) {
    const uint32_t p = wbase + 32u * i;
    ix[i] = p;
    img[i] = 0;
    if (p < E) {
      img[i] = T::ord(k0[bstart + p]);
      vor |= img[i];
      vand &= img[i];
    }
  }
  {
    const uint32_t lo_or = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)vor);
    const uint32_t lo_and = __reduce_and_sync(0xFFFFFFFFu, (uint32_t)vand);
    uint32_t hi_or = 0, hi_and = 0xFFFFFFFFu;
    if (sizeof(O) == 8) {
      hi_or = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)((uint64_t)vor >> 32));
      hi_and = __reduce_and_sync(0xFFFFFFFFu, (uint32_t)((uint64_t)vand >> 32));
    }
    if (lane == 0 && wbase < E) {
      atomicOr(&misc[0], lo_or);
      atomicAnd(&misc[2], lo_and);
      if (sizeof(O) == 8) { atomicOr(&misc[1], hi_or); atomicAnd(&misc[3], hi_and); }
    }
  }
  __syncthreads();
  if (warp == 0) {  // per-word prefix of unit starts; parity carried across words
    uint32_t carry = 0, pc = 0;
    for (uint32_t w0 = 0; w0 < nwords; w0 += 32) {
      const uint32_t w = w0 + lane;
      const uint32_t ub = w < nwords ? ubits[w] : 0u;
      const uint32_t c = (uint32_t)__popc(ub);
      uint32_t incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)lane >= o) incl += y;
      }
      if (w < nwords) upre[w] = carry + incl - c;
      carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
      const int hb = ub ? 31 - __clz(ub) : -1;
      const int own = hb >= 0 ? (int)((w < nwords ? pbits[w] : 0u) >> hb) & 1 : -1;
      const uint32_t has = __ballot_sync(0xFFFFFFFFu, own >= 0);
      const uint32_t le = has & (0xFFFFFFFFu >> (31 - lane));
      const int src = le ? 31 - __clz(le) : -1;
      const int ownv = __shfl_sync(0xFFFFFFFFu, own, src >= 0 ? src : 0);
      const uint32_t pw = src >= 0 ? (uint32_t)ownv : pc;
      if (w < nwords) pcar[w] = pw;
      pc = __shfl_sync(0xFFFFFFFFu, pw, 31);
    }
  }
  const uint64_t vary = ((uint64_t)(misc[1] ^ misc[3]) << 32) | (uint64_t)(misc[0] ^ misc[2]);
  __syncthreads();

  auto unit_of = [&](uint32_t q) -> uint32_t {
    const uint32_t w = q >> 5;
    return upre[w] + (uint32_t)__popc(ubits[w] & (0xFFFFFFFFu >> (31u - (q & 31u)))) - 1u;
  };

  // One stable counting pass on digit dg(i) (< 256): rank within the warp,
  // block-wide offsets (digit-major, then warp), scatter, striped reload.
  uint32_t cur = 0;
  uint32_t* const wc = cnt + warp * 256;
  auto pass = [&](auto digit) {
    for (uint32_t j = lane; j < 256; j += 32) wc[j] = 0u;
    __syncwarp();
    uint32_t rd[LR_ITEMS];  // rank | digit << 16
#pragma unroll
    for (int i = 0; i < LR_ITEMS; ++i) {
      const bool valid = wbase + 32u * i < E;
      const uint32_t vmask = __ballot_sync(0xFFFFFFFFu, valid);
      rd[i] = 0;
      if (valid) {
        const uint32_t d = digit(i);
        const uint32_t peers = __match_any_sync(vmask, d);
        const uint32_t leader = (uint32_t)__ffs(peers) - 1u;
        uint32_t base = 0;
        if (lane == leader) base = wc[d];
        base = __shfl_sync(vmask, base, leader);
        if (lane == leader) wc[d] = base + (uint32_t)__popc(peers);
        rd[i] = (base + (uint32_t)__popc(peers & lanemask_lt())) | (d << 16);
      }
      __syncwarp();
    }
    __syncthreads();
    if (tid < 256) {  // exclusive offsets of digit tid over the warps, then over digits
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < LR_WARPS; ++w) {
        const uint32_t c = cnt[w * 256 + tid];
        cnt[w * 256 + tid] = run;
        run += c;
      }
      uint32_t incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)lane >= o) incl += y;
      }
      if (lane == 31) misc[4 + warp] = incl;
      __syncwarp();
      asm volatile("bar.sync 1, 256;");
      uint32_t off = incl - run;
      for (uint32_t q = 0; q < warp; ++q) off += misc[4 + q];
#pragma unroll
      for (int w = 0; w < LR_WARPS; ++w) cnt[w * 256 + tid] += off;
    }
    __syncthreads();
    O* const dimg = simg + (cur ^ 1u) * LEAF_CAP;
    uint16_t* const didx = sidx + (cur ^ 1u) * LEAF_CAP;
#pragma unroll
    for (int i = 0; i < LR_ITEMS; ++i) {
      if (wbase + 32u * i < E) {
        const uint32_t pos = wc[rd[i] >> 16] + (rd[i] & 0xFFFFu);
        dimg[pos] = img[i];
        didx[pos] = (uint16_t)ix[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < LR_ITEMS; ++i) {
      const uint32_t p = wbase + 32u * i;
      if (p < E) { img[i] = dimg[p]; ix[i] = didx[p]; }
    }
    cur ^= 1u;
  };

  constexpr int KEY_BITS = 8 * (int)sizeof(O);
#pragma unroll 1
  for (int s = 0; s < KEY_BITS; s += 8) {
    if (((vary >> s) & 0xFFull) == 0) continue;  // this digit is equal over the batch
    pass([&](int i) -> uint32_t { return (uint32_t)(img[i] >> s) & 0xFFu; });
  }
#pragma unroll 1
  for (int s = 0; s < 16 && ((nunits - 1) >> s) != 0; s += 8) {
    pass([&](int i) -> uint32_t { return (unit_of(ix[i]) >> s) & 0xFFu; });
  }

  // write out: each unit to its parity buffer; gather payloads (and f32 key
  // bits: the order image maps all NaNs to one value) before any store, since
  // parity-0 units are written in place
  uint32_t gv[LR_ITEMS];
  K gk[LR_ITEMS];
#pragma unroll
  for (int i = 0; i < LR_ITEMS; ++i) {
    const uint32_t p = wbase + 32u * i;
    gv[i] = 0;
    gk[i] = (K)img[i];
    if (p < E) {
      if (HV) gv[i] = v0[bstart + ix[i]];
      if (KT == VMPS_KEY_F32) gk[i] = k0[bstart + ix[i]];
    }
  }
  if (HV || KT == VMPS_KEY_F32) __syncthreads();
#pragma unroll
  for (int i = 0; i < LR_ITEMS; ++i) {
    const uint32_t q = wbase + 32u * i;
    if (q < E) {
      const uint32_t w = q >> 5;
      const uint32_t mk = ubits[w] & (0xFFFFFFFFu >> (31u - (q & 31u)));
      const uint32_t par = mk ? (pbits[w] >> (31 - __clz(mk))) & 1u : pcar[w - 1];
      if (par) { k1[bstart + q] = gk[i]; if (HV) v1[bstart + q] = gv[i]; }
      else { k0[bstart + q] = gk[i]; if (HV) v0[bstart + q] = gv[i]; }
    }
  }
}

}  // namespace vmps
