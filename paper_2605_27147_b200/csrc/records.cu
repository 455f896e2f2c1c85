// records.cu -- large records (the paper's randomBlob30 /
// zeroBlob30 / ptr data types): n records of `words` u32 each,
// ordered lexicographically (unsigned words, word 0 most significant), sorted
// stably.  The records themselves move once: the engine sorts (key, u32
// index) pairs and one gather kernel writes the permuted records.
//
// Keys are 64-bit word pairs (w, w + 1).  The deciding pair f is the first
// one not equal in every record (pair 0 unless it is constant; then one scan
// finds the constant pairs).  One stable sort by pair f; if no two adjacent
// sorted keys are equal, or every later pair is constant, that order is the
// lexicographic one.  Otherwise the order is rebuilt LSD-style from the
// input order: one stable pass per non-constant word pair from the last to
// f (keys gathered through the current permutation) -- a stable sort by a
// constant key is the identity.  randomBlob30 and zeroBlob30 take one sort.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/vmps.h"

namespace {

thread_local std::string r_err;

__global__ void k_rec_iota(uint32_t* __restrict__ idx, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    idx[i] = (uint32_t)i;
}

// key[i] = (word w << 32) | word w+1 of record idx[i] (the missing word of an
// odd tail is 0); flags[0] |= any key differs from key[0]
__global__ void k_rec_pair_key(const uint32_t* __restrict__ rec, uint32_t words, uint32_t w,
                               const uint32_t* __restrict__ idx, uint64_t* __restrict__ key, uint64_t n,
                               uint32_t* __restrict__ flags) {
  const uint64_t k0 = ((uint64_t)rec[w] << 32) | (w + 1 < words ? rec[w + 1] : 0u);  // record 0 is in every permutation
  bool diff = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* r = rec + (uint64_t)idx[i] * words;
    const uint64_t k = ((uint64_t)r[w] << 32) | (w + 1 < words ? r[w + 1] : 0u);
    key[i] = k;
    diff |= k != k0;
  }
  if (__any_sync(0xFFFFFFFFu, diff) && (threadIdx.x & 31u) == 0) atomicOr(flags, 1u);
}

// mask |= bit q for every word pair q (< 64) that differs from record 0's
__global__ void k_rec_const_pairs(const uint32_t* __restrict__ rec, uint32_t words, uint64_t n,
                                  unsigned long long* __restrict__ mask) {
  const uint32_t np = min((words + 1) / 2, 64u);
  unsigned long long m = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* r = rec + i * words;
    for (uint32_t w = 0; w < 2 * np && w < words; ++w)
      if (r[w] != rec[w]) m |= 1ull << (w / 2);
  }
  for (int o = 16; o; o >>= 1) m |= __shfl_xor_sync(0xFFFFFFFFu, m, o);
  if ((threadIdx.x & 31u) == 0 && m) atomicOr(mask, m);
}

// flags[1] |= some adjacent keys are equal
__global__ void k_rec_ties(const uint64_t* __restrict__ key, uint64_t n, uint32_t* __restrict__ flags) {
  bool tie = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x)
    tie |= key[i] == key[i + 1];
  if (__any_sync(0xFFFFFFFFu, tie) && (threadIdx.x & 31u) == 0) atomicOr(flags + 1, 1u);
}

// out[i] = rec[idx[i]]: one thread per word, so both sides are contiguous runs
// of `words` words (reads gathered per record, writes fully coalesced)
__global__ void k_rec_gather(const uint32_t* __restrict__ rec, const uint32_t* __restrict__ idx, uint32_t words,
                             uint32_t* __restrict__ out, uint64_t total) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = t / words, w = t - i * words;
    out[t] = rec[(uint64_t)idx[i] * words + w];
  }
}

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

unsigned grid(uint64_t items) {
  const uint64_t g = (items + 255) / 256;
  return (unsigned)(g < 148u * 16u ? (g ? g : 1) : 148u * 16u);
}

#define RK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      r_err = std::string(#call) + ": " + cudaGetErrorString(e_);              \
      return VMPS_ERR_CUDA;                                                    \
    }                                                                          \
  } while (0)
#define RV(call)                                                               \
  do {                                                                         \
    vmps_status_t v_ = (call);                                                 \
    if (v_ != VMPS_OK) {                                                       \
      r_err = std::string(#call) + ": " + vmps_last_error();                   \
      return v_;                                                               \
    }                                                                          \
  } while (0)

}  // namespace

extern "C" {

vmps_status_t vmps_sort_records_workspace_bytes(uint64_t n, uint32_t words, size_t* h_bytes) {
  if (!h_bytes || words == 0 || n > VMPS_MAX_N) return VMPS_ERR_INVALID_ARG;
  size_t sb = 0;
  if (n > 1 && vmps_workspace_bytes(n, VMPS_KEY_U64, 1, VMPS_SCRATCH_UNBOUNDED, &sb) != VMPS_OK)
    return VMPS_ERR_INVALID_ARG;
  *h_bytes = al(n * 4 + 16) + al(n * 8 + 16) + al(64) + al(sb) + 256;
  return VMPS_OK;
}

vmps_status_t vmps_sort_records(const uint32_t* records, uint32_t* records_out, uint32_t* perm_out, uint64_t n,
                                uint32_t words, void* ws, size_t ws_bytes, void* stream) {
  if (words == 0 || n > VMPS_MAX_N) { r_err = "need words >= 1 and n <= VMPS_MAX_N"; return VMPS_ERR_INVALID_ARG; }
  if (n && (!records || (!records_out && !perm_out))) { r_err = "NULL records / outputs"; return VMPS_ERR_INVALID_ARG; }
  if (records_out && records_out == records) { r_err = "records_out must not alias records"; return VMPS_ERR_INVALID_ARG; }
  if (n == 0) return VMPS_OK;
  size_t need = 0;
  RV(vmps_sort_records_workspace_bytes(n, words, &need));
  if (!ws || ws_bytes < need) { r_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  cudaStream_t s = (cudaStream_t)stream;
  char* base = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  uint32_t* idx = (uint32_t*)base;
  uint64_t* key = (uint64_t*)(base + al(n * 4 + 16));
  uint32_t* flags = (uint32_t*)(base + al(n * 4 + 16) + al(n * 8 + 16));
  void* sws = base + al(n * 4 + 16) + al(n * 8 + 16) + al(64);
  const size_t sws_bytes = need - (al(n * 4 + 16) + al(n * 8 + 16) + al(64) + 256);
  const unsigned g = grid(n);
  uint32_t hf[2] = {0, 0};
  const uint32_t npairs = (words + 1) / 2;
  unsigned long long* dmask = (unsigned long long*)(flags + 4);
  auto pair_key = [&](uint32_t q) -> vmps_status_t {  // key of word pair q through idx; hf[0] = not constant
    RK(cudaMemsetAsync(flags, 0, 8, s));
    k_rec_pair_key<<<g, 256, 0, s>>>(records, words, 2 * q, idx, key, n, flags);
    RK(cudaMemcpyAsync(hf, flags, 8, cudaMemcpyDeviceToHost, s));
    RK(cudaStreamSynchronize(s));
    return VMPS_OK;
  };
  k_rec_iota<<<g, 256, 0, s>>>(idx, n);
  // the deciding pair: the first one that is not equal in every record
  uint32_t f = 0;
  unsigned long long mask = ~0ull;  // non-constant pairs (bit q), all unknown = set
  bool known = false;
  RV(pair_key(0));
  if (!hf[0] && npairs > 1 && npairs <= 64) {
    RK(cudaMemsetAsync(dmask, 0, 8, s));
    k_rec_const_pairs<<<g, 256, 0, s>>>(records, words, n, dmask);
    RK(cudaMemcpyAsync(&mask, dmask, 8, cudaMemcpyDeviceToHost, s));
    RK(cudaStreamSynchronize(s));
    known = true;
    if (!mask) f = npairs;  // every record equal: the identity
    else {
      f = (uint32_t)__builtin_ctzll(mask);
      RV(pair_key(f));
    }
  } else if (!hf[0] && npairs > 64) {
    // many words: no constant-pair scan, LSD below decides
    f = 0;
  }
  if (f < npairs && n > 1) {
    if (hf[0]) RV(vmps_sort_pairs(key, idx, n, VMPS_KEY_U64, VMPS_SCRATCH_UNBOUNDED, sws, sws_bytes, s, nullptr));
    // later pairs matter only if some record pair ties on pair f
    const bool later = known ? (mask >> (f + 1)) != 0ull : f + 1 < npairs;
    if (later) {
      RK(cudaMemsetAsync(flags + 1, 0, 4, s));
      k_rec_ties<<<g, 256, 0, s>>>(key, n, flags);
      RK(cudaMemcpyAsync(hf, flags, 8, cudaMemcpyDeviceToHost, s));
      RK(cudaStreamSynchronize(s));
      if (hf[1]) {
        // LSD over the non-constant pairs from the last to f, from the input order
        k_rec_iota<<<g, 256, 0, s>>>(idx, n);
        for (int64_t q = (int64_t)npairs - 1; q >= (int64_t)f; --q) {
          if (known && q < 64 && !((mask >> q) & 1ull)) continue;  // constant pair: identity
          RV(pair_key((uint32_t)q));
          if (!hf[0]) continue;
          RV(vmps_sort_pairs(key, idx, n, VMPS_KEY_U64, VMPS_SCRATCH_UNBOUNDED, sws, sws_bytes, s, nullptr));
        }
      }
    }
  }
  if (records_out) {
    const uint64_t total = n * words;
    k_rec_gather<<<grid(total), 256, 0, s>>>(records, idx, words, records_out, total);
  }
  if (perm_out) RK(cudaMemcpyAsync(perm_out, idx, n * 4, cudaMemcpyDeviceToDevice, s));
  RK(cudaGetLastError());
  return VMPS_OK;
}

const char* vmps_records_last_error(void) { return r_err.c_str(); }

}  // extern "C"
