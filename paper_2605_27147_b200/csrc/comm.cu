// comm.cu -- native multi-GPU entry points: one call per
// rank, NCCL over NVLink / NVSwitch for the exchange steps.
//
//   vmps_sort_*_dist      contiguous shards -> local sort -> exact splitters
//                         (16-ary search over the key order image, counts by
//                         vmps_count_rank summed with ncclAllReduce) -> grouped
//                         ncclSend / ncclRecv of the pieces -> stable merge of
//                         the received pieces in source-rank order.  In place:
//                         rank p ends with global output ranks [off_p, off_p +
//                         n_p), off_p = sum of the earlier shards' sizes.
//   vmps_merge_plan_dist  Alg. 1's plan of the concatenated shards (reading
//                         C13): per-shard chain transfer tables, all-gathered
//                         and composed from START(0); per-shard run emission;
//                         run lists broadcast to every rank; powers / tree /
//                         order on the whole run list; each rank keeps its
//                         runs and the merges whose boundary j is in its shard.
//
// Every data-path step runs in libvmps kernels (the public entry points of
// api.cu); this file holds the protocol, the host-side composition and the
// NCCL calls.  NCCL is loaded with dlopen on first use (the process's
// libnccl.so.2, e.g. the one torch already loaded), so the library has no
// link-time NCCL dependency.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cub/device/device_select.cuh>

#include "../../include/vmps.h"

namespace {

thread_local std::string c_err;

struct Nccl {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};
Nccl g_nccl;

bool nccl_load() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { c_err = "NCCL not found (dlopen libnccl.so.2)"; return false; }
  bool ok = true;
  auto sym = [&](const char* name) { void* p = dlsym(h, name); if (!p) ok = false; return p; };
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))sym("ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))sym("ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))sym("ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))sym("ncclAllReduce");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))sym("ncclAllGather");
  g_nccl.Broadcast = (decltype(g_nccl.Broadcast))sym("ncclBroadcast");
  g_nccl.Send = (decltype(g_nccl.Send))sym("ncclSend");
  g_nccl.Recv = (decltype(g_nccl.Recv))sym("ncclRecv");
  g_nccl.GroupStart = (decltype(g_nccl.GroupStart))sym("ncclGroupStart");
  g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))sym("ncclGroupEnd");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))sym("ncclGetErrorString");
  if (!ok) { c_err = "NCCL library lacks a required symbol"; return false; }
  g_nccl.ok = true;
  return true;
}

#define NC(call)                                                               \
  do {                                                                         \
    ncclResult_t r_ = (call);                                                  \
    if (r_ != ncclSuccess) {                                                   \
      c_err = std::string(#call) + ": " + g_nccl.GetErrorString(r_);           \
      return VMPS_ERR_NCCL;                                                    \
    }                                                                          \
  } while (0)
#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      c_err = std::string(#call) + ": " + cudaGetErrorString(e_);              \
      return VMPS_ERR_CUDA;                                                    \
    }                                                                          \
  } while (0)
#define VK(call)                                                               \
  do {                                                                         \
    vmps_status_t v_ = (call);                                                 \
    if (v_ != VMPS_OK) {                                                       \
      c_err = std::string(#call) + ": " + vmps_last_error();                   \
      return v_;                                                               \
    }                                                                          \
  } while (0)

size_t kbytes(vmps_key_t kt) { return kt == VMPS_KEY_U64 ? 8 : 4; }
size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

uint32_t minrun_of(uint64_t n) {
  uint64_t l = n;
  while (l >= 64) l = (l + 1) / 2;
  return (uint32_t)std::max<uint64_t>(l, 1);
}

// Bump allocator over the caller's workspace.
struct Carve {
  char* base;
  size_t off = 0, cap;
  Carve(void* ws, size_t bytes) : base((char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255)), cap(bytes) {
    cap = ws ? bytes - (size_t)(base - (char*)ws) : 0;
  }
  void* take(size_t b) {
    void* p = base + off;
    off += al(b);
    return off <= cap ? p : nullptr;
  }
};

// Gather one int64 value (or a fixed-size vector) from every rank into host memory.
template <typename T>
vmps_status_t gather_host(vmps_comm_t c, const T* h_mine, size_t count, std::vector<T>* out, T* d_buf,
                          cudaStream_t s);

}  // namespace

struct vmps_comm_s {
  ncclComm_t nc;
  int rank, world, device;
};

namespace {

template <typename T>
vmps_status_t gather_host(vmps_comm_t c, const T* h_mine, size_t count, std::vector<T>* out, T* d_buf,
                          cudaStream_t s) {
  // d_buf holds (world + 1) * count elements: own slot at the end, gathered at the front
  T* mine = d_buf + (size_t)c->world * count;
  CK(cudaMemcpyAsync(mine, h_mine, count * sizeof(T), cudaMemcpyHostToDevice, s));
  NC(g_nccl.AllGather(mine, d_buf, count * sizeof(T), ncclUint8, c->nc, s));
  out->resize((size_t)c->world * count);
  CK(cudaMemcpyAsync(out->data(), d_buf, out->size() * sizeof(T), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return VMPS_OK;
}

uint64_t img_max(vmps_key_t kt) { return kt == VMPS_KEY_U64 ? ~0ull : 0xFFFFFFFFull; }

// Per-rank cut for output rank R given every rank's counts of '< v*' and
// '<= v*' (v* = least v with sum(le) >= R): all elements < v*, then the tie
// group at v* in rank order (stability) -- as dist.split_points.
std::vector<uint64_t> split_points(uint64_t R, const std::vector<uint64_t>& lt, const std::vector<uint64_t>& le) {
  uint64_t sum_lt = 0;
  for (uint64_t x : lt) sum_lt += x;
  int64_t need = (int64_t)R - (int64_t)sum_lt;
  std::vector<uint64_t> cuts(lt.size());
  for (size_t q = 0; q < lt.size(); ++q) {
    const int64_t eq = (int64_t)(le[q] - lt[q]);
    const int64_t take = std::min<int64_t>(std::max<int64_t>(need, 0), eq);
    cuts[q] = lt[q] + (uint64_t)take;
    need -= take;
  }
  return cuts;
}

struct DistLayout {
  size_t sort_ws, mr_ws, recv_k, recv_v, probes, small, total;
};

DistLayout dist_layout(uint64_t n_local, vmps_key_t kt, int has_vals, int world, int64_t scratch) {
  DistLayout L{};
  size_t b = 0;
  vmps_workspace_bytes(std::max<uint64_t>(n_local, 1), kt, has_vals, scratch, &b);
  L.sort_ws = al(b);
  b = 0;
  vmps_merge_runs_workspace_bytes(std::max<uint64_t>(n_local, 1), kt, has_vals, (uint32_t)world, &b);
  L.mr_ws = al(b);
  L.recv_k = al(n_local * kbytes(kt) + 16);
  L.recv_v = has_vals ? al(n_local * 4 + 16) : 0;
  const size_t nprobe = (size_t)15 * std::max(world - 1, 1);
  L.probes = al(nprobe * 8) + 2 * al(nprobe * 8) + al(2 * nprobe * 8);
  L.small = al(((size_t)world + 1) * std::max<size_t>(64, 2 * (size_t)world) * 8);
  L.total = std::max(L.sort_ws, L.mr_ws) + L.recv_k + L.recv_v + L.probes + L.small + 256;
  return L;
}

vmps_status_t sort_dist_any(vmps_comm_t c, void* keys, uint32_t* vals, uint64_t n_local, vmps_key_t kt,
                            int64_t scratch, void* ws, size_t ws_bytes, cudaStream_t s, vmps_stats_t* h_stats) {
  if (!c) { c_err = "NULL communicator"; return VMPS_ERR_INVALID_ARG; }
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) {
    c_err = "unknown key type";
    return VMPS_ERR_INVALID_ARG;
  }
  const int g = c->world, me = c->rank;
  const int hv = vals ? 1 : 0;
  const DistLayout L = dist_layout(n_local, kt, hv, g, scratch);
  if (!ws || ws_bytes < L.total) { c_err = "workspace too small (vmps_dist_workspace_bytes)"; return VMPS_ERR_BUDGET; }
  Carve cv(ws, ws_bytes);
  void* sort_ws = cv.take(std::max(L.sort_ws, L.mr_ws));
  void* rk = cv.take(L.recv_k);
  uint32_t* rv = hv ? (uint32_t*)cv.take(L.recv_v) : nullptr;
  const size_t nprobe_cap = (size_t)15 * std::max(g - 1, 1);
  uint64_t* d_probe = (uint64_t*)cv.take(nprobe_cap * 8);
  uint64_t* d_lt = (uint64_t*)cv.take(nprobe_cap * 8);
  uint64_t* d_le = (uint64_t*)cv.take(nprobe_cap * 8);
  uint64_t* d_cnt = (uint64_t*)cv.take(2 * nprobe_cap * 8);
  uint64_t* d_small = (uint64_t*)cv.take(L.small);
  if (!d_small) { c_err = "workspace carve"; return VMPS_ERR_BUDGET; }
  // 1. shard sizes and output ranks
  std::vector<uint64_t> sizes;
  VK(gather_host<uint64_t>(c, &n_local, 1, &sizes, d_small, s));
  std::vector<uint64_t> off(g + 1, 0);
  for (int q = 0; q < g; ++q) off[q + 1] = off[q] + sizes[q];
  // 2. local sort
  if (n_local > 1) {
    if (hv) VK(vmps_sort_pairs(keys, vals, n_local, kt, scratch, sort_ws, std::max(L.sort_ws, L.mr_ws), s, h_stats));
    else VK(vmps_sort_keys(keys, n_local, kt, scratch, sort_ws, std::max(L.sort_ws, L.mr_ws), s, h_stats));
  }
  if (g == 1) return VMPS_OK;
  // 3. exact splitters for R_t = off_t, t = 1..g-1: 16-ary search over the image
  const int m = g - 1;
  std::vector<uint64_t> lo(m, 0), hi(m, img_max(kt));
  std::vector<uint64_t> probe, le_h(nprobe_cap);
  for (;;) {
    probe.clear();
    std::vector<int> base(m + 1, 0);
    for (int t = 0; t < m; ++t) {
      base[t] = (int)probe.size();
      if (lo[t] < hi[t]) {
        const uint64_t w = hi[t] - lo[t];
        for (int k = 1; k <= 15; ++k) {  // strictly inside [lo, hi): lo + k w / 16 (distinct, increasing)
          const uint64_t pr = lo[t] + (uint64_t)(((unsigned __int128)w * k) / 16);
          if (probe.size() > (size_t)base[t] && probe.back() >= pr) continue;
          if (pr >= hi[t]) break;
          probe.push_back(pr);
        }
        if (probe.size() == (size_t)base[t]) probe.push_back(lo[t]);
      }
    }
    base[m] = (int)probe.size();
    if (probe.empty()) break;
    CK(cudaMemcpyAsync(d_probe, probe.data(), probe.size() * 8, cudaMemcpyHostToDevice, s));
    if (n_local) VK(vmps_count_rank(keys, n_local, kt, d_probe, (uint32_t)probe.size(), d_lt, d_le, s));
    else CK(cudaMemsetAsync(d_le, 0, probe.size() * 8, s));
    NC(g_nccl.AllReduce(d_le, d_le, probe.size(), ncclUint64, ncclSum, c->nc, s));
    CK(cudaMemcpyAsync(le_h.data(), d_le, probe.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int t = 0; t < m; ++t) {
      if (!(lo[t] < hi[t])) continue;
      const uint64_t R = off[t + 1];
      // least probe with #(<= probe) >= R bounds v* from above; the probe
      // before it (#(<= p) < R) from below
      uint64_t nlo = lo[t], nhi = hi[t];
      for (int k = base[t]; k < base[t + 1]; ++k) {
        if (le_h[k] >= R) { nhi = probe[k]; break; }
        nlo = probe[k] + 1;
      }
      lo[t] = nlo;
      hi[t] = std::max(nlo, nhi);
    }
  }
  // final counts at v* on every rank
  for (int t = 0; t < m; ++t) probe.push_back(lo[t]);
  CK(cudaMemcpyAsync(d_probe, probe.data(), (size_t)m * 8, cudaMemcpyHostToDevice, s));
  if (n_local) VK(vmps_count_rank(keys, n_local, kt, d_probe, (uint32_t)m, d_cnt, d_cnt + m, s));
  else CK(cudaMemsetAsync(d_cnt, 0, 2 * (size_t)m * 8, s));
  std::vector<uint64_t> allc;
  {
    std::vector<uint64_t> mine(2 * (size_t)m);
    CK(cudaMemcpyAsync(mine.data(), d_cnt, 2 * (size_t)m * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    VK(gather_host<uint64_t>(c, mine.data(), 2 * (size_t)m, &allc, d_small, s));
  }
  // cut[q][t]: elements of rank q that go to ranks < t
  std::vector<std::vector<uint64_t>> cut(g, std::vector<uint64_t>(g + 1, 0));
  for (int q = 0; q < g; ++q) cut[q][g] = sizes[q];
  for (int t = 0; t < m; ++t) {
    std::vector<uint64_t> lt(g), le(g);
    for (int q = 0; q < g; ++q) {
      lt[q] = allc[(size_t)q * 2 * m + t];
      le[q] = allc[(size_t)q * 2 * m + m + t];
    }
    const std::vector<uint64_t> pts = split_points(off[t + 1], lt, le);
    for (int q = 0; q < g; ++q) cut[q][t + 1] = pts[q];
  }
  // 4. exchange: piece [cut[me][p], cut[me][p+1]) to rank p; receive in rank order
  const size_t kb = kbytes(kt);
  std::vector<uint64_t> roff(g + 1, 0);
  for (int q = 0; q < g; ++q) roff[q + 1] = roff[q] + (cut[q][me + 1] - cut[q][me]);
  if (roff[g] != n_local) { c_err = "internal: received count differs from the shard size"; return VMPS_ERR_INTERNAL; }
  NC(g_nccl.GroupStart());
  for (int p = 0; p < g; ++p) {
    const uint64_t sn = cut[me][p + 1] - cut[me][p];
    const uint64_t rn = roff[p + 1] - roff[p];
    if (sn) {
      NC(g_nccl.Send((const char*)keys + cut[me][p] * kb, sn * kb, ncclUint8, p, c->nc, s));
      if (hv) NC(g_nccl.Send(vals + cut[me][p], sn * 4, ncclUint8, p, c->nc, s));
    }
    if (rn) {
      NC(g_nccl.Recv((char*)rk + roff[p] * kb, rn * kb, ncclUint8, p, c->nc, s));
      if (hv) NC(g_nccl.Recv(rv + roff[p], rn * 4, ncclUint8, p, c->nc, s));
    }
  }
  NC(g_nccl.GroupEnd());
  // 5. stable merge of the received pieces (ties to the lower source rank)
  std::vector<uint64_t> starts;
  for (int q = 0; q < g; ++q)
    if (roff[q + 1] > roff[q]) starts.push_back(roff[q]);
  if (starts.size() > 1)
    VK(vmps_merge_runs(rk, rv, n_local, kt, starts.data(), (uint32_t)starts.size(), sort_ws,
                       std::max(L.sort_ws, L.mr_ws), s));
  if (n_local) {
    CK(cudaMemcpyAsync(keys, rk, n_local * kb, cudaMemcpyDeviceToDevice, s));
    if (hv) CK(cudaMemcpyAsync(vals, rv, n_local * 4, cudaMemcpyDeviceToDevice, s));
  }
  return VMPS_OK;
}

// ---- distributed merge plan ----
struct InShard {
  uint64_t lo, hi;
  __host__ __device__ __forceinline__ bool operator()(const vmps_merge_rec_t& r) const {
    return r.j >= lo && r.j < hi;
  }
};

struct PlanLayout {
  size_t shard_ws, plan_ws, edges, tabs, runs, kinds, recs, sel_tmp, small, total;
};

PlanLayout plan_layout(uint64_t n_total, uint64_t n_local, vmps_key_t kt, int world) {
  PlanLayout L{};
  const uint32_t mr = minrun_of(n_total);
  const uint32_t H = mr + 8;
  size_t b = 0;
  if (n_local) vmps_shard_workspace_bytes(n_local, kt, mr, &b);
  L.shard_ws = al(b);
  const uint64_t rcap = n_total / mr + 2 * (uint64_t)world + 2;
  b = 0;
  vmps_plan_workspace_bytes(rcap, &b);
  L.plan_ws = al(b);
  L.edges = al(((size_t)world + 1) * (H + 1) * kbytes(kt)) + al(H * kbytes(kt) + 16);
  L.tabs = al(((size_t)world + 1) * 3 * mr * 8);
  L.runs = al((rcap + 1) * 8);
  L.kinds = al(rcap + 16);
  L.recs = al(rcap * sizeof(vmps_merge_rec_t));
  size_t tmp = 0;
  cub::DeviceSelect::If(nullptr, tmp, (vmps_merge_rec_t*)nullptr, (uint64_t*)nullptr, (int64_t)rcap, InShard{0, 0});
  L.sel_tmp = al(tmp + 16);
  L.small = al(((size_t)world + 1) * 64 * 8);
  L.total = std::max(L.shard_ws, L.plan_ws) + L.edges + L.tabs + L.runs + L.kinds + L.recs + L.sel_tmp + L.small + 256;
  return L;
}

}  // namespace

extern "C" {

vmps_status_t vmps_comm_unique_id(void* h_id128) {
  if (!h_id128) return VMPS_ERR_INVALID_ARG;
  if (!nccl_load()) return VMPS_ERR_NCCL;
  ncclUniqueId id;
  NC(g_nccl.GetUniqueId(&id));
  memcpy(h_id128, &id, sizeof(id));
  return VMPS_OK;
}

vmps_status_t vmps_comm_init(vmps_comm_t* h_out, int rank, int world, const void* h_id128, int device) {
  if (!h_out || !h_id128 || world < 1 || rank < 0 || rank >= world) return VMPS_ERR_INVALID_ARG;
  if (!nccl_load()) return VMPS_ERR_NCCL;
  CK(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, h_id128, sizeof(id));
  vmps_comm_s* c = new vmps_comm_s{nullptr, rank, world, device};
  ncclResult_t r = g_nccl.CommInitRank(&c->nc, world, id, rank);
  if (r != ncclSuccess) {
    c_err = std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r);
    delete c;
    return VMPS_ERR_NCCL;
  }
  *h_out = c;
  return VMPS_OK;
}

vmps_status_t vmps_comm_destroy(vmps_comm_t c) {
  if (!c) return VMPS_OK;
  ncclResult_t r = g_nccl.ok ? g_nccl.CommDestroy(c->nc) : ncclSuccess;
  delete c;
  if (r != ncclSuccess) { c_err = "ncclCommDestroy failed"; return VMPS_ERR_NCCL; }
  return VMPS_OK;
}

const char* vmps_comm_last_error(void) { return c_err.c_str(); }

// ---- peer mappings for the pull-merge (CUDA IPC over NVLink) ----
vmps_status_t vmps_ipc_handle(const void* d_ptr, void* h_handle64, uint64_t* h_offset) {
  if (!d_ptr || !h_handle64 || !h_offset) return VMPS_ERR_INVALID_ARG;
  // the handle names the whole allocation holding d_ptr; the peer adds the offset
  static CUresult (*get_range)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
  if (!get_range) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      c_err = "cuMemGetAddressRange unavailable";
      return VMPS_ERR_CUDA;
    }
    get_range = (CUresult(*)(CUdeviceptr*, size_t*, CUdeviceptr))fn;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)d_ptr) != CUDA_SUCCESS) { c_err = "cuMemGetAddressRange failed"; return VMPS_ERR_CUDA; }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, (void*)base));
  memcpy(h_handle64, &h, sizeof(h));
  *h_offset = (uint64_t)((CUdeviceptr)d_ptr - base);
  return VMPS_OK;
}

vmps_status_t vmps_ipc_open(const void* h_handle64, uint64_t offset, void** h_ptr) {
  if (!h_handle64 || !h_ptr) return VMPS_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle64, sizeof(h));
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *h_ptr = (char*)p + offset;
  return VMPS_OK;
}

vmps_status_t vmps_ipc_close(void* d_ptr, uint64_t offset) {
  if (!d_ptr) return VMPS_OK;
  CK(cudaIpcCloseMemHandle((char*)d_ptr - offset));
  return VMPS_OK;
}

vmps_status_t vmps_dist_workspace_bytes(uint64_t n_local, vmps_key_t kt, int has_vals, int world,
                                        int64_t scratch_elems, size_t* h_bytes) {
  if (!h_bytes || world < 1 || n_local > VMPS_MAX_N) return VMPS_ERR_INVALID_ARG;
  *h_bytes = dist_layout(n_local, kt, has_vals ? 1 : 0, world, scratch_elems).total;
  return VMPS_OK;
}

vmps_status_t vmps_sort_keys_dist(vmps_comm_t c, void* keys, uint64_t n_local, vmps_key_t kt, int64_t scratch_elems,
                                  void* ws, size_t ws_bytes, void* stream, vmps_stats_t* h_stats) {
  return sort_dist_any(c, keys, nullptr, n_local, kt, scratch_elems, ws, ws_bytes, (cudaStream_t)stream, h_stats);
}

vmps_status_t vmps_sort_pairs_dist(vmps_comm_t c, void* keys, uint32_t* vals, uint64_t n_local, vmps_key_t kt,
                                   int64_t scratch_elems, void* ws, size_t ws_bytes, void* stream,
                                   vmps_stats_t* h_stats) {
  if (!vals) { c_err = "vals is NULL (use vmps_sort_keys_dist)"; return VMPS_ERR_INVALID_ARG; }
  return sort_dist_any(c, keys, vals, n_local, kt, scratch_elems, ws, ws_bytes, (cudaStream_t)stream, h_stats);
}

vmps_status_t vmps_merge_plan_dist_workspace_bytes(uint64_t n_total, uint64_t n_local, vmps_key_t kt, int world,
                                                   size_t* h_bytes) {
  if (!h_bytes || world < 1 || n_local > n_total || n_local > VMPS_MAX_N) return VMPS_ERR_INVALID_ARG;
  *h_bytes = plan_layout(n_total, n_local, kt, world).total;
  return VMPS_OK;
}

vmps_status_t vmps_merge_plan_dist(vmps_comm_t c, const void* keys, uint64_t n_local, vmps_key_t kt,
                                   uint64_t* run_start, uint8_t* run_kind, vmps_merge_rec_t* merges,
                                   uint64_t cap_runs, uint64_t* h_num_runs_local, uint64_t* h_num_merges_local,
                                   void* ws, size_t ws_bytes, void* stream) {
  if (!c || !h_num_runs_local || !h_num_merges_local) return VMPS_ERR_INVALID_ARG;
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) return VMPS_ERR_INVALID_ARG;
  if (n_local > VMPS_MAX_N) { c_err = "n_local > VMPS_MAX_N"; return VMPS_ERR_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  const int g = c->world, me = c->rank;
  const size_t kb = kbytes(kt);
  // sizes -> offsets, n, minrun (workspace is checked once n is known)
  uint64_t* d_small0 = nullptr;
  {
    // the size exchange needs (g + 1) u64 of device memory before the carve
    Carve pre(ws, ws_bytes);
    d_small0 = (uint64_t*)pre.take(((size_t)g + 1) * 64 * 8);
    if (!d_small0) { c_err = "workspace too small"; return VMPS_ERR_BUDGET; }
  }
  std::vector<uint64_t> sizes;
  VK(gather_host<uint64_t>(c, &n_local, 1, &sizes, d_small0, s));
  std::vector<uint64_t> off(g + 1, 0);
  for (int q = 0; q < g; ++q) off[q + 1] = off[q] + sizes[q];
  const uint64_t N = off[g];
  if (N == 0) { *h_num_runs_local = *h_num_merges_local = 0; return VMPS_OK; }
  const PlanLayout L = plan_layout(N, n_local, kt, g);
  if (!ws || ws_bytes < L.total) { c_err = "workspace too small (vmps_merge_plan_dist_workspace_bytes)"; return VMPS_ERR_BUDGET; }
  Carve cv(ws, ws_bytes);
  uint64_t* d_small = (uint64_t*)cv.take(L.small);  // same place as d_small0
  void* shard_ws = cv.take(std::max(L.shard_ws, L.plan_ws));
  const uint32_t mr = minrun_of(N), H = mr + 8, ns = 3 * mr;
  char* d_edges = (char*)cv.take(((size_t)g + 1) * (H + 1) * kb);
  char* d_halo = (char*)cv.take(H * kb + 16);
  uint64_t* d_tabs = (uint64_t*)cv.take(((size_t)g + 1) * ns * 8);
  const uint64_t rcap = N / mr + 2 * (uint64_t)g + 2;
  uint64_t* d_runs = (uint64_t*)cv.take((rcap + 1) * 8);
  uint8_t* d_kinds = (uint8_t*)cv.take(rcap + 16);
  vmps_merge_rec_t* d_recs = (vmps_merge_rec_t*)cv.take(rcap * sizeof(vmps_merge_rec_t));
  void* d_sel = cv.take(L.sel_tmp);
  if (!d_sel) { c_err = "workspace carve"; return VMPS_ERR_BUDGET; }
  // edge keys: every shard's first H keys (zero padded) and its last key
  const size_t eb = (size_t)(H + 1) * kb;
  char* mine = d_edges + (size_t)g * eb;
  CK(cudaMemsetAsync(mine, 0, eb, s));
  const uint64_t h = std::min<uint64_t>(H, n_local);
  if (h) {
    CK(cudaMemcpyAsync(mine, keys, h * kb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(mine + (size_t)H * kb, (const char*)keys + (n_local - 1) * kb, kb, cudaMemcpyDeviceToDevice, s));
  }
  NC(g_nccl.AllGather(mine, d_edges, eb, ncclUint8, c->nc, s));
  int pq = -1;
  for (int q = me - 1; q >= 0; --q)
    if (sizes[q]) { pq = q; break; }
  const void* d_prev = pq >= 0 ? (const void*)(d_edges + (size_t)pq * eb + (size_t)H * kb) : nullptr;
  uint32_t nh = 0;  // halo: the next H keys of the global array, from the following shards' heads
  for (int q = me + 1; q < g && nh < H; ++q) {
    const uint32_t take = (uint32_t)std::min<uint64_t>(sizes[q], H - nh);
    if (take) CK(cudaMemcpyAsync(d_halo + (size_t)nh * kb, d_edges + (size_t)q * eb, (size_t)take * kb,
                                 cudaMemcpyDeviceToDevice, s));
    nh += take;
  }
  const uint64_t rem = N - off[me];
  const uint32_t n_end = rem >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)rem;
  // transfer tables -> entry states and run counts
  uint64_t* tmine = d_tabs + (size_t)g * ns;
  if (n_local)
    VK(vmps_shard_chain(keys, n_local, kt, mr, n_end, d_prev, nh ? d_halo : nullptr, nh, tmine, shard_ws,
                        std::max(L.shard_ws, L.plan_ws), s));
  else
    CK(cudaMemsetAsync(tmine, 0, (size_t)ns * 8, s));
  NC(g_nccl.AllGather(tmine, d_tabs, (size_t)ns * 8, ncclUint8, c->nc, s));
  std::vector<uint64_t> tabs((size_t)g * ns);
  CK(cudaMemcpyAsync(tabs.data(), d_tabs, tabs.size() * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<uint64_t> cnt(g, 0);
  std::vector<uint32_t> entry(g, 0);
  uint32_t st = 0;  // START(0)
  for (int q = 0; q < g; ++q) {
    entry[q] = st;
    if (!sizes[q] || st == 255u) continue;
    const uint64_t v = tabs[(size_t)q * ns + st];
    cnt[q] = v & 0xFFFFFFFFull;
    st = (uint32_t)(v >> 32);
  }
  std::vector<uint64_t> roff(g + 1, 0);
  for (int q = 0; q < g; ++q) roff[q + 1] = roff[q] + cnt[q];
  const uint64_t r = roff[g];
  if (r > rcap) { c_err = "internal: run capacity"; return VMPS_ERR_INTERNAL; }
  if (cnt[me])
    VK(vmps_shard_runs(keys, n_local, kt, mr, n_end, d_prev, nh ? d_halo : nullptr, nh, entry[me], cnt[me], off[me],
                       d_runs + roff[me], d_kinds + roff[me], shard_ws, std::max(L.shard_ws, L.plan_ws), s));
  // every rank's run list to every rank, in place, rank order
  NC(g_nccl.GroupStart());
  for (int q = 0; q < g; ++q) {
    if (!cnt[q]) continue;
    NC(g_nccl.Broadcast(d_runs + roff[q], d_runs + roff[q], cnt[q], ncclUint64, q, c->nc, s));
    NC(g_nccl.Broadcast(d_kinds + roff[q], d_kinds + roff[q], cnt[q], ncclUint8, q, c->nc, s));
  }
  NC(g_nccl.GroupEnd());
  CK(cudaMemcpyAsync(d_runs + r, &N, 8, cudaMemcpyHostToDevice, s));
  // this rank's runs
  if (cnt[me] > cap_runs) { c_err = "cap_runs too small"; *h_num_runs_local = cnt[me]; return VMPS_ERR_INVALID_ARG; }
  if (cnt[me]) {
    if (!run_start || !run_kind) return VMPS_ERR_INVALID_ARG;
    CK(cudaMemcpyAsync(run_start, d_runs + roff[me], cnt[me] * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(run_kind, d_kinds + roff[me], cnt[me], cudaMemcpyDeviceToDevice, s));
  }
  *h_num_runs_local = cnt[me];
  // the whole plan, then the merges whose boundary j lies in this shard
  uint64_t nm = 0;
  if (r >= 2) {
    VK(vmps_plan_from_runs(d_runs, r, N, d_recs, shard_ws, std::max(L.shard_ws, L.plan_ws), s));
    uint64_t* d_nsel = d_small;
    size_t tmp = L.sel_tmp;
    CK(cub::DeviceSelect::If(d_sel, tmp, d_recs, d_nsel, (int64_t)(r - 1), InShard{off[me], off[me] + n_local}, s));
    CK(cudaMemcpyAsync(&nm, d_nsel, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (nm > cap_runs) { c_err = "cap_runs too small for the merges"; *h_num_merges_local = nm; return VMPS_ERR_INVALID_ARG; }
    if (nm) {
      if (!merges) return VMPS_ERR_INVALID_ARG;
      CK(cudaMemcpyAsync(merges, d_recs, nm * sizeof(vmps_merge_rec_t), cudaMemcpyDeviceToDevice, s));
    }
  }
  *h_num_merges_local = nm;
  CK(cudaStreamSynchronize(s));
  return VMPS_OK;
}

}  // extern "C"
