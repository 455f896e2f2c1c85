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
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_select.cuh>
#include <nvtx3/nvToolsExt.h>

#include "../../include/vmps.h"

namespace {

thread_local std::string c_err;

struct Nccl {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommAbort)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
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
std::mutex g_nccl_mu;

bool nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
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
  g_nccl.CommAbort = (decltype(g_nccl.CommAbort))sym("ncclCommAbort");
  g_nccl.CommGetAsyncError = (decltype(g_nccl.CommGetAsyncError))sym("ncclCommGetAsyncError");
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
      if (v_ != VMPS_ERR_NCCL || c_err.empty())                                \
        c_err = std::string(#call) + ": " + vmps_last_error() + " " + c_err;   \
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

double comm_timeout_s() {
  const char* e = getenv("VMPS_COMM_TIMEOUT_S");
  const double t = e ? atof(e) : 0.0;
  return t > 0 ? t : 600.0;
}

// ---------------------------------------------------------------------------
// In-process group of virtual ranks (threads of one process, any devices):
// the same protocol as NCCL, with collectives made of host barriers, CUDA
// events and device-to-device copies.  Lets tests run the library's own
// multi-rank protocol with g ranks on one GPU (NCCL refuses two
// ranks on one device).
// ---------------------------------------------------------------------------
constexpr int LG_MAXW = 256;
struct LocalGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  double timeout_s;
  // per-rank published state of the current collective
  const void* ptr[LG_MAXW];
  size_t bytes[LG_MAXW];
  std::vector<std::vector<std::pair<const void*, size_t>>> sends;  // [src][dst]
  std::vector<std::vector<std::pair<const void*, size_t>>> bc;     // [rank][item]
  cudaEvent_t ev_ready[LG_MAXW], ev_done[LG_MAXW];
  uint64_t* tmp[LG_MAXW];  // per-rank reduction scratch (device)
  size_t tmp_cap = 0;
};

}  // namespace

struct vmps_comm_s {
  int kind;  // 0 NCCL, 1 in-process virtual ranks
  ncclComm_t nc;
  LocalGroup* lg;
  int rank, world, device;
  bool aborted;
};

namespace {

// barrier of the local group; false on timeout (the group is then broken)
bool lg_barrier(LocalGroup* g) {
  std::unique_lock<std::mutex> lk(g->m);
  if (g->broken) return false;
  const uint64_t my = g->gen;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return true;
  }
  const bool ok = g->cv.wait_for(lk, std::chrono::duration<double>(g->timeout_s),
                                 [&] { return g->gen != my || g->broken; });
  if (!ok || g->broken) {
    g->broken = true;
    g->cv.notify_all();
    return false;
  }
  return true;
}

#define LB(g)                                                                  \
  do {                                                                         \
    if (!lg_barrier(g)) {                                                      \
      c_err = "virtual-rank group: barrier timeout or a rank failed";          \
      return VMPS_ERR_NCCL;                                                    \
    }                                                                          \
  } while (0)

// Phase helpers of a local collective: inputs ready -> copies -> done.
vmps_status_t lg_begin(vmps_comm_t c, cudaStream_t s) {
  LocalGroup* g = c->lg;
  CK(cudaEventRecord(g->ev_ready[c->rank], s));
  LB(g);
  for (int q = 0; q < g->world; ++q)
    if (q != c->rank) CK(cudaStreamWaitEvent(s, g->ev_ready[q], 0));
  return VMPS_OK;
}
vmps_status_t lg_end(vmps_comm_t c, cudaStream_t s) {
  LocalGroup* g = c->lg;
  CK(cudaEventRecord(g->ev_done[c->rank], s));
  LB(g);
  for (int q = 0; q < g->world; ++q)
    if (q != c->rank) CK(cudaStreamWaitEvent(s, g->ev_done[q], 0));
  return VMPS_OK;
}

__global__ void k_sum_u64(uint64_t* out, const uint64_t* const* src, int world, size_t count) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    uint64_t a = 0;
    for (int q = 0; q < world; ++q) a += src[q][i];
    out[i] = a;
  }
}

// ---- transport: the collectives the protocols use ----
// in-place sum of count u64 over all ranks
vmps_status_t tp_allreduce_u64(vmps_comm_t c, uint64_t* d, size_t count, cudaStream_t s) {
  if (c->kind == 0) {
    NC(g_nccl.AllReduce(d, d, count, ncclUint64, ncclSum, c->nc, s));
    return VMPS_OK;
  }
  LocalGroup* g = c->lg;
  if ((count + (size_t)g->world) * 8 > g->tmp_cap) {
    c_err = "virtual-rank group: reduction too large";
    return VMPS_ERR_INTERNAL;
  }
  g->ptr[c->rank] = d;
  VK(lg_begin(c, s));
  // the source pointer table travels as a kernel argument array in device scratch
  uint64_t* tmp = g->tmp[c->rank];
  const uint64_t** tab = (const uint64_t**)(tmp + count);
  std::vector<const uint64_t*> hp(g->world);
  for (int q = 0; q < g->world; ++q) hp[q] = (const uint64_t*)g->ptr[q];
  CK(cudaMemcpyAsync(tab, hp.data(), g->world * sizeof(void*), cudaMemcpyHostToDevice, s));
  k_sum_u64<<<1, 256, 0, s>>>(tmp, tab, g->world, count);
  CK(cudaGetLastError());
  VK(lg_end(c, s));  // every rank has read every d
  CK(cudaMemcpyAsync(d, tmp, count * 8, cudaMemcpyDeviceToDevice, s));
  return VMPS_OK;  // (the pageable host table was staged by the copy call)
}

// d_all[q * bytes ..] = rank q's d_mine
vmps_status_t tp_allgather(vmps_comm_t c, const void* d_mine, void* d_all, size_t bytes, cudaStream_t s) {
  if (c->kind == 0) {
    NC(g_nccl.AllGather(d_mine, d_all, bytes, ncclUint8, c->nc, s));
    return VMPS_OK;
  }
  LocalGroup* g = c->lg;
  g->ptr[c->rank] = d_mine;
  VK(lg_begin(c, s));
  for (int q = 0; q < g->world; ++q)
    if (bytes) CK(cudaMemcpyAsync((char*)d_all + (size_t)q * bytes, g->ptr[q], bytes, cudaMemcpyDeviceToDevice, s));
  return lg_end(c, s);
}

struct BItem { void* d; size_t bytes; int root; };
// in-place broadcasts (item i from its root to every rank; same item list on all ranks)
vmps_status_t tp_bcast_many(vmps_comm_t c, const std::vector<BItem>& items, cudaStream_t s) {
  if (c->kind == 0) {
    NC(g_nccl.GroupStart());
    for (const BItem& b : items) NC(g_nccl.Broadcast(b.d, b.d, b.bytes, ncclUint8, b.root, c->nc, s));
    NC(g_nccl.GroupEnd());
    return VMPS_OK;
  }
  LocalGroup* g = c->lg;
  auto& mine = g->bc[c->rank];
  mine.clear();
  for (const BItem& b : items) mine.push_back({b.d, b.bytes});
  VK(lg_begin(c, s));
  for (size_t i = 0; i < items.size(); ++i) {
    const BItem& b = items[i];
    if (b.root != c->rank && b.bytes)
      CK(cudaMemcpyAsync(b.d, g->bc[b.root][i].first, b.bytes, cudaMemcpyDeviceToDevice, s));
  }
  return lg_end(c, s);
}

struct P2P { int peer; const void* p; size_t bytes; };
// grouped point-to-point: sends[i] to sends[i].peer, recvs[i] from recvs[i].peer;
// at most one send per (peer, tag) order: the k-th send to a peer pairs with
// the peer's k-th receive from this rank
vmps_status_t tp_exchange(vmps_comm_t c, const std::vector<P2P>& sends, const std::vector<P2P>& recvs,
                          cudaStream_t s) {
  if (c->kind == 0) {
    NC(g_nccl.GroupStart());
    for (const P2P& x : sends) NC(g_nccl.Send(x.p, x.bytes, ncclUint8, x.peer, c->nc, s));
    for (const P2P& x : recvs) NC(g_nccl.Recv((void*)x.p, x.bytes, ncclUint8, x.peer, c->nc, s));
    NC(g_nccl.GroupEnd());
    return VMPS_OK;
  }
  LocalGroup* g = c->lg;
  auto& mine = g->sends[c->rank];
  mine.clear();
  for (const P2P& x : sends) mine.push_back({x.p, (size_t)x.peer | ((size_t)x.bytes << 8)});
  VK(lg_begin(c, s));
  // match the k-th receive from q with q's k-th send to this rank
  std::vector<int> seen(g->world, 0);
  for (const P2P& x : recvs) {
    int k = seen[x.peer]++, hit = -1;
    const auto& sq = g->sends[x.peer];
    for (size_t i = 0; i < sq.size(); ++i)
      if ((int)(sq[i].second & 0xFF) == c->rank && k-- == 0) { hit = (int)i; break; }
    if (hit < 0 || (sq[hit].second >> 8) != x.bytes) {
      c_err = "virtual-rank group: unmatched send / receive (rank " + std::to_string(c->rank) + " from " +
              std::to_string(x.peer) + ", " + std::to_string(x.bytes) + " bytes; the peer posted " +
              std::to_string(sq.size()) + " sends" +
              (sq.empty() ? std::string() : ", first " + std::to_string(sq[0].second >> 8) + " bytes to " +
                                                std::to_string(sq[0].second & 0xFF)) + ")";
      return VMPS_ERR_INTERNAL;
    }
    if (x.bytes) CK(cudaMemcpyAsync((void*)x.p, sq[hit].first, x.bytes, cudaMemcpyDeviceToDevice, s));
  }
  return lg_end(c, s);
}

// Wait for the stream, polling NCCL's asynchronous error state and a timeout
// (VMPS_COMM_TIMEOUT_S, default 600 s): a failed or stuck peer returns
// VMPS_ERR_NCCL (the communicator is aborted) instead of hanging.
vmps_status_t tp_sync(vmps_comm_t c, cudaStream_t s) {
  const auto t0 = std::chrono::steady_clock::now();
  const double lim = comm_timeout_s();
  for (int it = 0;; ++it) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return VMPS_OK;
    if (e != cudaErrorNotReady) {
      c_err = std::string("stream: ") + cudaGetErrorString(e);
      return VMPS_ERR_CUDA;
    }
    if (c->kind == 0 && !c->aborted) {
      ncclResult_t ar = ncclSuccess;
      if (g_nccl.CommGetAsyncError(c->nc, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
        c_err = std::string("NCCL asynchronous error: ") + g_nccl.GetErrorString(ar);
        g_nccl.CommAbort(c->nc);
        c->aborted = true;
        return VMPS_ERR_NCCL;
      }
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > lim) {
      c_err = "communication timeout (VMPS_COMM_TIMEOUT_S)";
      if (c->kind == 0 && !c->aborted) { g_nccl.CommAbort(c->nc); c->aborted = true; }
      return VMPS_ERR_NCCL;
    }
    if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// Gather a fixed-size vector of u64 from every rank into host memory.
vmps_status_t gather_host(vmps_comm_t c, const uint64_t* h_mine, size_t count, std::vector<uint64_t>* out,
                          uint64_t* d_buf, cudaStream_t s) {
  // d_buf holds (world + 1) * count elements: own slot at the end, gathered at the front
  uint64_t* mine = d_buf + (size_t)c->world * count;
  CK(cudaMemcpyAsync(mine, h_mine, count * 8, cudaMemcpyHostToDevice, s));
  VK(tp_allgather(c, mine, d_buf, count * 8, s));
  out->resize((size_t)c->world * count);
  CK(cudaMemcpyAsync(out->data(), d_buf, out->size() * 8, cudaMemcpyDeviceToHost, s));
  return tp_sync(c, s);
}

uint64_t img_max(vmps_key_t kt) { return kt == VMPS_KEY_U64 ? ~0ull : 0xFFFFFFFFull; }

// ---------------------------------------------------------------------------
// Host-side protocol arithmetic (exported below for the Python path and the
// CPU tests; no device work).
// ---------------------------------------------------------------------------
constexpr uint32_t SPLIT_ARITY = 16;  // probes per splitter per round: 15

// probes of one search round for the m splitters still open (lo < hi):
// lo + k (hi - lo) / 16, k = 1..15, strictly increasing inside [lo, hi)
void splitter_probes(uint32_t m, const uint64_t* lo, const uint64_t* hi, std::vector<uint64_t>* probe,
                     std::vector<uint32_t>* base) {
  probe->clear();
  base->assign(m + 1, 0);
  for (uint32_t t = 0; t < m; ++t) {
    (*base)[t] = (uint32_t)probe->size();
    if (lo[t] < hi[t]) {
      const uint64_t w = hi[t] - lo[t];
      for (uint32_t k = 1; k < SPLIT_ARITY; ++k) {
        const uint64_t pr = lo[t] + (uint64_t)(((unsigned __int128)w * k) / SPLIT_ARITY);
        if (probe->size() > (*base)[t] && probe->back() >= pr) continue;
        if (pr >= hi[t]) break;
        probe->push_back(pr);
      }
      if (probe->size() == (*base)[t]) probe->push_back(lo[t]);
    }
  }
  (*base)[m] = (uint32_t)probe->size();
}

// v*_t = the least image value v with #{x <= v} >= R_t: the least probe with
// sum(le) >= R bounds it from above, the probe before it from below
void splitter_update(uint32_t m, uint64_t* lo, uint64_t* hi, const uint64_t* R, const uint64_t* probe,
                     const uint32_t* base, const uint64_t* le_sum) {
  for (uint32_t t = 0; t < m; ++t) {
    if (!(lo[t] < hi[t])) continue;
    uint64_t nlo = lo[t], nhi = hi[t];
    for (uint32_t k = base[t]; k < base[t + 1]; ++k) {
      if (le_sum[k] >= R[t]) { nhi = probe[k]; break; }
      nlo = probe[k] + 1;
    }
    lo[t] = nlo;
    hi[t] = std::max(nlo, nhi);
  }
}

// Per-rank cut for output rank R given every rank's counts of '< v*' and
// '<= v*' (v* = least v with sum(le) >= R): all elements < v*, then the tie
// group at v* in rank order (lower ranks first: the stable sort of the
// concatenation, P:657's tie rule across shards).
void split_points(uint32_t g, uint64_t R, const uint64_t* lt, const uint64_t* le, uint64_t* cuts) {
  uint64_t sum_lt = 0;
  for (uint32_t q = 0; q < g; ++q) sum_lt += lt[q];
  int64_t need = (int64_t)R - (int64_t)sum_lt;
  for (uint32_t q = 0; q < g; ++q) {
    const int64_t eq = (int64_t)(le[q] - lt[q]);
    const int64_t take = std::min<int64_t>(std::max<int64_t>(need, 0), eq);
    cuts[q] = lt[q] + (uint64_t)take;
    need -= take;
  }
}

// Chain composition of the shards' run-detection transfer tables from
// START(0): entry state and runs started per shard (empty shards are the
// identity; END = 255 stops the chain).
void compose_tables(uint32_t g, uint32_t ns, const uint64_t* tabs, const uint64_t* sizes, uint32_t* entry,
                    uint64_t* count) {
  uint32_t st = 0;
  for (uint32_t q = 0; q < g; ++q) {
    entry[q] = st;
    count[q] = 0;
    if (!sizes[q] || st == 255u) continue;
    const uint64_t v = tabs[(size_t)q * ns + st];
    count[q] = v & 0xFFFFFFFFull;
    st = (uint32_t)(v >> 32);
  }
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

// Steps 1-3 of the distributed sort on sorted shards: shard sizes and exact
// splitters; cut[q * (g + 1) + t] = elements of rank q that go to ranks < t.
vmps_status_t dist_cuts(vmps_comm_t c, const void* keys, uint64_t n_local, vmps_key_t kt, uint64_t* d_probe,
                        uint64_t* d_lt, uint64_t* d_le, uint64_t* d_cnt, uint64_t* d_small, size_t nprobe_cap,
                        cudaStream_t s, std::vector<uint64_t>* sizes_out, std::vector<uint64_t>* cut_out,
                        uint32_t* rounds_out) {
  const int g = c->world;
  std::vector<uint64_t> sizes;
  VK(gather_host(c, &n_local, 1, &sizes, d_small, s));
  std::vector<uint64_t> off(g + 1, 0);
  for (int q = 0; q < g; ++q) off[q + 1] = off[q] + sizes[q];
  std::vector<uint64_t> cut((size_t)g * (g + 1), 0);
  for (int q = 0; q < g; ++q) cut[(size_t)q * (g + 1) + g] = sizes[q];
  uint32_t rounds = 0;
  if (g > 1) {
    const uint32_t m = (uint32_t)g - 1;
    std::vector<uint64_t> lo(m, 0), hi(m, img_max(kt)), R(m), probe, le_h(nprobe_cap);
    std::vector<uint32_t> base;
    for (uint32_t t = 0; t < m; ++t) R[t] = off[t + 1];
    for (;;) {
      splitter_probes(m, lo.data(), hi.data(), &probe, &base);
      if (probe.empty()) break;
      ++rounds;
      CK(cudaMemcpyAsync(d_probe, probe.data(), probe.size() * 8, cudaMemcpyHostToDevice, s));
      if (n_local) VK(vmps_count_rank(keys, n_local, kt, d_probe, (uint32_t)probe.size(), d_lt, d_le, s));
      else CK(cudaMemsetAsync(d_le, 0, probe.size() * 8, s));
      VK(tp_allreduce_u64(c, d_le, probe.size(), s));
      CK(cudaMemcpyAsync(le_h.data(), d_le, probe.size() * 8, cudaMemcpyDeviceToHost, s));
      VK(tp_sync(c, s));
      splitter_update(m, lo.data(), hi.data(), R.data(), probe.data(), base.data(), le_h.data());
    }
    // final counts at v* on every rank
    CK(cudaMemcpyAsync(d_probe, lo.data(), (size_t)m * 8, cudaMemcpyHostToDevice, s));
    if (n_local) VK(vmps_count_rank(keys, n_local, kt, d_probe, m, d_cnt, d_cnt + m, s));
    else CK(cudaMemsetAsync(d_cnt, 0, 2 * (size_t)m * 8, s));
    std::vector<uint64_t> mine(2 * (size_t)m), allc;
    CK(cudaMemcpyAsync(mine.data(), d_cnt, 2 * (size_t)m * 8, cudaMemcpyDeviceToHost, s));
    VK(tp_sync(c, s));
    VK(gather_host(c, mine.data(), 2 * (size_t)m, &allc, d_small, s));
    std::vector<uint64_t> lt(g), le(g), pts(g);
    for (uint32_t t = 0; t < m; ++t) {
      for (int q = 0; q < g; ++q) {
        lt[q] = allc[(size_t)q * 2 * m + t];
        le[q] = allc[(size_t)q * 2 * m + m + t];
      }
      split_points((uint32_t)g, off[t + 1], lt.data(), le.data(), pts.data());
      for (int q = 0; q < g; ++q) cut[(size_t)q * (g + 1) + t + 1] = pts[q];
    }
  }
  if (sizes_out) *sizes_out = sizes;
  if (cut_out) *cut_out = cut;
  if (rounds_out) *rounds_out = rounds;
  return VMPS_OK;
}

// A rank that fails outside a collective breaks its virtual-rank group, so
// the other ranks return promptly instead of waiting for the timeout.
vmps_status_t fail_group(vmps_comm_t c, vmps_status_t rc) {
  if (rc != VMPS_OK && c && c->kind == 1) {
    std::lock_guard<std::mutex> lk(c->lg->m);
    c->lg->broken = true;
    c->lg->cv.notify_all();
  }
  return rc;
}

// ---------------------------------------------------------------------------
// Scratch-bounded distributed sort (second half): every
// rank's extra element memory stays within its cap S (c sqrt(n log n) per GPU,
// exchange staging included).  There is no receive buffer: after the local
// scratch-bounded sort, adjacent ranks repeat stable merge-splits
// (odd-even transposition over the rank order).  In a merge-split of ranks
// a < b = a + 1 holding sorted A and B, the pair finds by the same 16-ary
// search the cut c = #A among the first |A| outputs of the stable merge of A B
// (ties to A); a's tail A[c, |A|) and b's head B[0, |A| - c) swap
// places in chunks of S/2 elements through staging (out + in = S), and each
// rank then holds two sorted runs, merged by its local scratch-bounded sort.
// Each step is a stable merge of two adjacent segments of the rank-ordered
// sequence, so equal keys never change their relative order; phases repeat
// until an even and an odd phase swap nothing, i.e. every adjacent pair is in
// order: the unique stable sort of the concatenation, each rank keeping its
// element count.
// ---------------------------------------------------------------------------
struct BdLayout {
  size_t sort_ws, stage, small, total;
  uint64_t C;  // staging chunk (elements)
};

BdLayout bd_layout(uint64_t n_local, vmps_key_t kt, int hv, int world, int64_t S) {
  BdLayout L{};
  size_t b = 0, b2 = 0;
  vmps_workspace_bytes(std::max<uint64_t>(n_local, 1), kt, hv, S, &b);
  vmps_merge_runs_bounded_workspace_bytes(std::max<uint64_t>(n_local, 1), kt, hv, 2, S, &b2);
  b = std::max(b, b2);
  L.C = std::max<uint64_t>(1, (uint64_t)S / 2);
  const size_t w = kbytes(kt) + (hv ? 4 : 0);
  L.stage = al(2 * L.C * w + 64);
  L.sort_ws = al(b);
  L.small = al(((size_t)world * 16 + 64) * 8) * 3;
  L.total = std::max(L.sort_ws, L.stage) + L.small + 256;  // staging overlays the sort's workspace
  return L;
}

// k_copy_u8: plain device copy within one stream (chunks of the swap)
vmps_status_t d2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
  return VMPS_OK;
}

vmps_status_t sort_dist_bounded(vmps_comm_t c, void* keys, uint32_t* vals, uint64_t n_local, vmps_key_t kt,
                                int64_t S, void* ws, size_t ws_bytes, cudaStream_t s, vmps_stats_t* h_stats,
                                bool pairs) {
  const int g = c->world, me = c->rank;
  const int hv = pairs ? 1 : 0;
  const size_t kb = kbytes(kt);
  const BdLayout L = bd_layout(n_local, kt, hv, g, S);
  if (!ws || ws_bytes < L.total) { c_err = "workspace too small (vmps_dist_workspace_bytes)"; return VMPS_ERR_BUDGET; }
  Carve cv(ws, ws_bytes);
  char* big = (char*)cv.take(std::max(L.sort_ws, L.stage));
  uint64_t* d_vec = (uint64_t*)cv.take(L.small / 3);
  uint64_t* d_probe = (uint64_t*)cv.take(L.small / 3);
  uint64_t* d_cnt = (uint64_t*)cv.take(L.small / 3);
  if (!d_cnt) { c_err = "workspace carve"; return VMPS_ERR_BUDGET; }
  const size_t big_bytes = std::max(L.sort_ws, L.stage);
  auto local_sort = [&](vmps_stats_t* st) -> vmps_status_t {
    if (n_local <= 1) return VMPS_OK;
    if (hv) return vmps_sort_pairs(keys, vals, n_local, kt, S, big, big_bytes, s, st);
    return vmps_sort_keys(keys, n_local, kt, S, big, big_bytes, s, st);
  };
  VK(local_sort(h_stats));
  if (g == 1) return VMPS_OK;
  std::vector<uint64_t> sizes;
  VK(gather_host(c, &n_local, 1, &sizes, d_vec, s));
  const size_t NV = (size_t)g * 16 + 2;  // per pair (slot = lower rank): 15 probe counts; + flags
  std::vector<uint64_t> h_vec(NV), h_probe;
  // the transposition runs over the non-empty ranks in rank order (an empty
  // rank holds nothing to order and just joins the collectives)
  std::vector<int> ne;
  int my_pos = -1;
  for (int q = 0; q < g; ++q)
    if (sizes[q]) {
      if (q == me) my_pos = (int)ne.size();
      ne.push_back(q);
    }
  // equal shards (BASELINE.json's configs) converge within g phases (block
  // odd-even transposition); unequal ones need more, since a merge-split moves
  // at most the smaller shard across a rank: the limit grows with max / min
  uint64_t nmin = ~0ull, nmax = 0;
  for (int q : ne) { nmin = std::min(nmin, sizes[q]); nmax = std::max(nmax, sizes[q]); }
  const int max_phase = ne.empty() ? 2 : (int)std::min<uint64_t>(1u << 20, (uint64_t)g + 8 + 2 * ((nmax + nmin - 1) / nmin));
  int quiet = 0;
  for (int phase = 0; quiet < 2 && phase < max_phase; ++phase) {
    int partner = -1;
    if (my_pos >= 0) {
      const int pp = ((my_pos + phase) % 2 == 0) ? my_pos + 1 : my_pos - 1;
      if (pp >= 0 && pp < (int)ne.size()) partner = ne[pp];
    }
    const bool paired = partner >= 0;
    const int lower = paired ? std::min(me, partner) : -1;
    const int upper = paired ? std::max(me, partner) : -1;
    const uint64_t nA = paired ? sizes[lower] : 0, nB = paired ? sizes[upper] : 0;
    // splitter v*: the least image with #(A <= v) + #(B <= v) >= |A|
    uint64_t lo = 0, hi = img_max(kt);
    bool open = paired && nA > 0 && nB > 0;
    for (;;) {
      std::vector<uint32_t> base;
      std::vector<uint64_t> pr;
      if (open) splitter_probes(1, &lo, &hi, &pr, &base);
      const bool active = open && !pr.empty();
      std::fill(h_vec.begin(), h_vec.end(), 0);
      h_vec[NV - 1] = active ? 1 : 0;
      CK(cudaMemcpyAsync(d_vec, h_vec.data(), NV * 8, cudaMemcpyHostToDevice, s));
      if (active && n_local) {
        CK(cudaMemcpyAsync(d_probe, pr.data(), pr.size() * 8, cudaMemcpyHostToDevice, s));
        VK(vmps_count_rank(keys, n_local, kt, d_probe, (uint32_t)pr.size(), d_cnt, d_vec + (size_t)lower * 16, s));
      }
      VK(tp_allreduce_u64(c, d_vec, NV, s));
      CK(cudaMemcpyAsync(h_vec.data(), d_vec, NV * 8, cudaMemcpyDeviceToHost, s));
      VK(tp_sync(c, s));
      if (h_vec[NV - 1] == 0) break;  // no pair is still searching
      if (active) {
        const uint64_t R[1] = {nA};
        splitter_update(1, &lo, &hi, R, pr.data(), base.data(), h_vec.data() + (size_t)lower * 16);
        open = lo < hi;
      }
    }
    // both partners' counts at v* -> the cut of A, the swap length, the chunk rounds
    std::fill(h_vec.begin(), h_vec.end(), 0);
    uint64_t lt = 0, le = 0;
    if (paired && nA > 0 && nB > 0 && n_local) {
      CK(cudaMemcpyAsync(d_probe, &lo, 8, cudaMemcpyHostToDevice, s));
      VK(vmps_count_rank(keys, n_local, kt, d_probe, 1, d_cnt, d_cnt + 1, s));
      uint64_t two[2];
      CK(cudaMemcpyAsync(two, d_cnt, 16, cudaMemcpyDeviceToHost, s));
      VK(tp_sync(c, s));
      lt = two[0];
      le = two[1];
      const size_t o = (size_t)lower * 16 + (me == lower ? 0 : 2);
      h_vec[o] = lt;
      h_vec[o + 1] = le;
    }
    if (paired) h_vec[(size_t)lower * 16 + 4 + (me == lower ? 0 : 1)] = L.C;  // each side's staging chunk
    CK(cudaMemcpyAsync(d_vec, h_vec.data(), NV * 8, cudaMemcpyHostToDevice, s));
    VK(tp_allreduce_u64(c, d_vec, NV, s));
    CK(cudaMemcpyAsync(h_vec.data(), d_vec, NV * 8, cudaMemcpyDeviceToHost, s));
    VK(tp_sync(c, s));
    uint64_t cnt = 0;
    if (paired && nA > 0 && nB > 0) {
      const uint64_t* q = h_vec.data() + (size_t)lower * 16;
      const uint64_t ltv[2] = {q[0], q[2]}, lev[2] = {q[1], q[3]};
      uint64_t cut[2];
      split_points(2, nA, ltv, lev, cut);
      cnt = nA - cut[0];  // A's tail that moves up = B's head that moves down
    }
    // the pair swaps in chunks both staging buffers hold (the caps may differ)
    const uint64_t C = paired ? std::max<uint64_t>(1, std::min(h_vec[(size_t)lower * 16 + 4],
                                                              h_vec[(size_t)lower * 16 + 5]))
                              : L.C;
    const uint64_t my_rounds = (cnt + C - 1) / C;
    // every rank runs the same number of exchange rounds (empty when done)
    std::fill(h_vec.begin(), h_vec.end(), 0);
    h_vec[(size_t)me] = my_rounds;
    h_vec[NV - 2] = cnt ? 1 : 0;
    CK(cudaMemcpyAsync(d_vec, h_vec.data(), NV * 8, cudaMemcpyHostToDevice, s));
    VK(tp_allreduce_u64(c, d_vec, NV, s));
    CK(cudaMemcpyAsync(h_vec.data(), d_vec, NV * 8, cudaMemcpyDeviceToHost, s));
    VK(tp_sync(c, s));
    uint64_t rounds = 0;
    for (int q = 0; q < g; ++q) rounds = std::max(rounds, h_vec[(size_t)q]);
    const bool swapped = h_vec[NV - 2] != 0;
    // my region of the swap: A[c, |A|) on the lower rank, B[0, cnt) on the upper
    const uint64_t r0 = (me == lower) ? nA - cnt : 0;
    char* sk_out = big;
    char* sk_in = big + C * kb;
    char* sv_out = big + 2 * C * kb;
    char* sv_in = sv_out + C * 4;
    for (uint64_t r = 0; r < rounds; ++r) {
      std::vector<P2P> sends, recvs;
      const uint64_t a = r * C, b = std::min(cnt, a + C);
      if (a < b) {
        const size_t m = b - a;
        VK(d2d(sk_out, (const char*)keys + (r0 + a) * kb, m * kb, s));
        sends.push_back({partner, sk_out, m * kb});
        recvs.push_back({partner, sk_in, m * kb});
        if (hv) {
          VK(d2d(sv_out, vals + r0 + a, m * 4, s));
          sends.push_back({partner, sv_out, m * 4});
          recvs.push_back({partner, sv_in, m * 4});
        }
      }
      VK(tp_exchange(c, sends, recvs, s));
      if (a < b) {
        const size_t m = b - a;
        VK(d2d((char*)keys + (r0 + a) * kb, sk_in, m * kb, s));
        if (hv) VK(d2d(vals + r0 + a, sv_in, m * 4, s));
      }
    }
    if (cnt) {  // two sorted runs -> one: the bounded merge of given runs (ties to the first run)
      const uint64_t runs[2] = {0, me == lower ? nA - cnt : cnt};
      if (hv) VK(vmps_merge_runs_bounded(keys, vals, n_local, kt, runs, 2, S, big, big_bytes, s));
      else VK(vmps_merge_runs_bounded(keys, nullptr, n_local, kt, runs, 2, S, big, big_bytes, s));
    }
    quiet = swapped ? 0 : quiet + 1;
  }
  if (quiet < 2) { c_err = "internal: merge-split phases did not converge"; return VMPS_ERR_INTERNAL; }
  if (h_stats) {  // the cap covers the exchange staging as well (it overlays the sort's scratch)
    h_stats->scratch_bytes = std::max<uint64_t>(h_stats->scratch_bytes, 2 * L.C * (kb + (hv ? 4 : 0)));
    h_stats->peak_extra_device_bytes = std::max<uint64_t>(h_stats->peak_extra_device_bytes, L.total);
  }
  return tp_sync(c, s);
}

vmps_status_t sort_dist_any(vmps_comm_t c, void* keys, uint32_t* vals, uint64_t n_local, vmps_key_t kt,
                            int64_t scratch, void* ws, size_t ws_bytes, cudaStream_t s, vmps_stats_t* h_stats,
                            bool pairs) {
  if (!c) { c_err = "NULL communicator"; return VMPS_ERR_INVALID_ARG; }
  if (scratch >= 0) {
    if (n_local && !keys) { c_err = "keys is NULL"; return VMPS_ERR_INVALID_ARG; }
    c_err.clear();
    return sort_dist_bounded(c, keys, vals, n_local, kt, scratch, ws, ws_bytes, s, h_stats, pairs);
  }
  if (n_local && !keys) { c_err = "keys is NULL"; return VMPS_ERR_INVALID_ARG; }
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) {
    c_err = "unknown key type";
    return VMPS_ERR_INVALID_ARG;
  }
  c_err.clear();
  const int g = c->world, me = c->rank;
  const int hv = pairs ? 1 : 0;  // (an empty shard may pass NULL buffers)
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
  struct Nv { explicit Nv(const char* m) { nvtxRangePushA(m); } ~Nv() { nvtxRangePop(); } } nv("vmps_sort_dist");
  // 1. local sort
  if (n_local > 1) {
    if (hv) VK(vmps_sort_pairs(keys, vals, n_local, kt, scratch, sort_ws, std::max(L.sort_ws, L.mr_ws), s, h_stats));
    else VK(vmps_sort_keys(keys, n_local, kt, scratch, sort_ws, std::max(L.sort_ws, L.mr_ws), s, h_stats));
  }
  if (g == 1) return VMPS_OK;
  // 2-3. shard sizes, exact splitters (16-ary search over the key order image)
  std::vector<uint64_t> sizes, cutv;
  VK(dist_cuts(c, keys, n_local, kt, d_probe, d_lt, d_le, d_cnt, d_small, nprobe_cap, s, &sizes, &cutv, nullptr));
  auto cut = [&](int q, int t) { return cutv[(size_t)q * (g + 1) + t]; };
  // 4. exchange: piece [cut(me, p), cut(me, p+1)) to rank p; receive in rank order
  const size_t kb = kbytes(kt);
  std::vector<uint64_t> roff(g + 1, 0);
  for (int q = 0; q < g; ++q) roff[q + 1] = roff[q] + (cut(q, me + 1) - cut(q, me));
  if (roff[g] != n_local) { c_err = "internal: received count differs from the shard size"; return VMPS_ERR_INTERNAL; }
  std::vector<P2P> sends, recvs;
  for (int p = 0; p < g; ++p) {
    const uint64_t sn = cut(me, p + 1) - cut(me, p);
    const uint64_t rn = roff[p + 1] - roff[p];
    if (sn) {
      sends.push_back({p, (const char*)keys + cut(me, p) * kb, sn * kb});
      if (hv) sends.push_back({p, vals + cut(me, p), sn * 4});
    }
    if (rn) {
      recvs.push_back({p, (char*)rk + roff[p] * kb, rn * kb});
      if (hv) recvs.push_back({p, rv + roff[p], rn * 4});
    }
  }
  VK(tp_exchange(c, sends, recvs, s));
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
  vmps_comm_s* c = new vmps_comm_s{0, nullptr, nullptr, rank, world, device, false};
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
  ncclResult_t r = ncclSuccess;
  if (c->kind == 0 && g_nccl.ok) r = c->aborted ? ncclSuccess : g_nccl.CommDestroy(c->nc);
  delete c;
  if (r != ncclSuccess) { c_err = "ncclCommDestroy failed"; return VMPS_ERR_NCCL; }
  return VMPS_OK;
}

vmps_status_t vmps_local_group_create(int world, int device, void** h_group) {
  if (!h_group || world < 1 || world > LG_MAXW) return VMPS_ERR_INVALID_ARG;
  CK(cudaSetDevice(device));
  LocalGroup* g = new LocalGroup();
  g->world = world;
  g->timeout_s = comm_timeout_s();
  g->sends.assign(world, {});
  g->bc.assign(world, {});
  g->tmp_cap = 64 * 1024;
  for (int q = 0; q < world; ++q) {
    g->ptr[q] = nullptr;
    g->bytes[q] = 0;
    if (cudaEventCreateWithFlags(&g->ev_ready[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_done[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc((void**)&g->tmp[q], g->tmp_cap) != cudaSuccess) {
      c_err = "virtual-rank group: CUDA resources";
      return VMPS_ERR_CUDA;
    }
  }
  *h_group = g;
  return VMPS_OK;
}

vmps_status_t vmps_local_group_destroy(void* group) {
  LocalGroup* g = (LocalGroup*)group;
  if (!g) return VMPS_OK;
  cudaDeviceSynchronize();
  for (int q = 0; q < g->world; ++q) {
    cudaEventDestroy(g->ev_ready[q]);
    cudaEventDestroy(g->ev_done[q]);
    cudaFree(g->tmp[q]);
  }
  delete g;
  return VMPS_OK;
}

vmps_status_t vmps_comm_init_local(vmps_comm_t* h_out, int rank, void* group, int device) {
  LocalGroup* g = (LocalGroup*)group;
  if (!h_out || !g || rank < 0 || rank >= g->world) return VMPS_ERR_INVALID_ARG;
  CK(cudaSetDevice(device));
  *h_out = new vmps_comm_s{1, nullptr, g, rank, g->world, device, false};
  return VMPS_OK;
}

vmps_status_t vmps_dist_cuts_workspace_bytes(int world, size_t* h_bytes) {
  if (!h_bytes || world < 1) return VMPS_ERR_INVALID_ARG;
  const size_t np = (size_t)15 * std::max(world - 1, 1);
  *h_bytes = 3 * al(np * 8) + al(2 * np * 8) + al(((size_t)world + 1) * std::max<size_t>(64, 2 * (size_t)world) * 8) + 256;
  return VMPS_OK;
}

vmps_status_t vmps_dist_cuts(vmps_comm_t c, const void* keys, uint64_t n_local, vmps_key_t kt, uint64_t* h_cut,
                             uint64_t* h_sizes, uint32_t* h_rounds, void* ws, size_t ws_bytes, void* stream) {
  if (!c || !h_cut || (n_local && !keys)) return VMPS_ERR_INVALID_ARG;
  if (kt != VMPS_KEY_U32 && kt != VMPS_KEY_U64 && kt != VMPS_KEY_F32) return VMPS_ERR_INVALID_ARG;
  size_t need = 0;
  vmps_dist_cuts_workspace_bytes(c->world, &need);
  if (!ws || ws_bytes < need) { c_err = "workspace too small (vmps_dist_cuts_workspace_bytes)"; return VMPS_ERR_BUDGET; }
  c_err.clear();
  const size_t np = (size_t)15 * std::max(c->world - 1, 1);
  Carve cv(ws, ws_bytes);
  uint64_t* d_probe = (uint64_t*)cv.take(np * 8);
  uint64_t* d_lt = (uint64_t*)cv.take(np * 8);
  uint64_t* d_le = (uint64_t*)cv.take(np * 8);
  uint64_t* d_cnt = (uint64_t*)cv.take(2 * np * 8);
  uint64_t* d_small = (uint64_t*)cv.take(((size_t)c->world + 1) * std::max<size_t>(64, 2 * (size_t)c->world) * 8);
  if (!d_small) { c_err = "workspace carve"; return VMPS_ERR_BUDGET; }
  std::vector<uint64_t> sizes, cut;
  uint32_t rounds = 0;
  const vmps_status_t rc = fail_group(c, dist_cuts(c, keys, n_local, kt, d_probe, d_lt, d_le, d_cnt, d_small, np,
                                                   (cudaStream_t)stream, &sizes, &cut, &rounds));
  if (rc != VMPS_OK) return rc;
  memcpy(h_cut, cut.data(), cut.size() * 8);
  if (h_sizes) memcpy(h_sizes, sizes.data(), sizes.size() * 8);
  if (h_rounds) *h_rounds = rounds;
  return VMPS_OK;
}

// ---- host-side protocol arithmetic (see the functions above) ----
vmps_status_t vmps_splitter_probes(uint32_t m, const uint64_t* h_lo, const uint64_t* h_hi, uint64_t* h_probe,
                                   uint32_t* h_base, uint32_t* h_nprobe) {
  if ((m && (!h_lo || !h_hi || !h_probe)) || !h_base || !h_nprobe) return VMPS_ERR_INVALID_ARG;
  std::vector<uint64_t> pr;
  std::vector<uint32_t> base;
  splitter_probes(m, h_lo, h_hi, &pr, &base);
  if (!pr.empty()) memcpy(h_probe, pr.data(), pr.size() * 8);
  memcpy(h_base, base.data(), base.size() * 4);
  *h_nprobe = (uint32_t)pr.size();
  return VMPS_OK;
}

vmps_status_t vmps_splitter_update(uint32_t m, uint64_t* h_lo, uint64_t* h_hi, const uint64_t* h_R,
                                   const uint64_t* h_probe, const uint32_t* h_base, const uint64_t* h_le_sum) {
  if (m && (!h_lo || !h_hi || !h_R || !h_base)) return VMPS_ERR_INVALID_ARG;
  splitter_update(m, h_lo, h_hi, h_R, h_probe, h_base, h_le_sum);
  return VMPS_OK;
}

vmps_status_t vmps_split_points(uint32_t g, uint64_t R, const uint64_t* h_lt, const uint64_t* h_le, uint64_t* h_cut) {
  if (!g || !h_lt || !h_le || !h_cut) return VMPS_ERR_INVALID_ARG;
  split_points(g, R, h_lt, h_le, h_cut);
  return VMPS_OK;
}

vmps_status_t vmps_compose_tables(uint32_t g, uint32_t ns, const uint64_t* h_tables, const uint64_t* h_sizes,
                                  uint32_t* h_entry, uint64_t* h_count) {
  if (!g || !h_tables || !h_sizes || !h_entry || !h_count) return VMPS_ERR_INVALID_ARG;
  compose_tables(g, ns, h_tables, h_sizes, h_entry, h_count);
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
  *h_bytes = scratch_elems >= 0 ? bd_layout(n_local, kt, has_vals ? 1 : 0, world, scratch_elems).total
                                 : dist_layout(n_local, kt, has_vals ? 1 : 0, world, scratch_elems).total;
  return VMPS_OK;
}

vmps_status_t vmps_sort_keys_dist(vmps_comm_t c, void* keys, uint64_t n_local, vmps_key_t kt, int64_t scratch_elems,
                                  void* ws, size_t ws_bytes, void* stream, vmps_stats_t* h_stats) {
  return fail_group(c, sort_dist_any(c, keys, nullptr, n_local, kt, scratch_elems, ws, ws_bytes, (cudaStream_t)stream,
                                     h_stats, false));
}

vmps_status_t vmps_sort_pairs_dist(vmps_comm_t c, void* keys, uint32_t* vals, uint64_t n_local, vmps_key_t kt,
                                   int64_t scratch_elems, void* ws, size_t ws_bytes, void* stream,
                                   vmps_stats_t* h_stats) {
  if (!vals && n_local) { c_err = "vals is NULL (use vmps_sort_keys_dist)"; return fail_group(c, VMPS_ERR_INVALID_ARG); }
  return fail_group(c, sort_dist_any(c, keys, vals, n_local, kt, scratch_elems, ws, ws_bytes, (cudaStream_t)stream,
                                     h_stats, true));
}

vmps_status_t vmps_merge_plan_dist_workspace_bytes(uint64_t n_total, uint64_t n_local, vmps_key_t kt, int world,
                                                   size_t* h_bytes) {
  if (!h_bytes || world < 1 || n_local > n_total || n_local > VMPS_MAX_N) return VMPS_ERR_INVALID_ARG;
  *h_bytes = plan_layout(n_total, n_local, kt, world).total;
  return VMPS_OK;
}

vmps_status_t vmps_merge_plan_dist_capacity(uint64_t n_total, uint64_t n_local, uint64_t* h_cap) {
  if (!h_cap || n_local > n_total) return VMPS_ERR_INVALID_ARG;
  // runs starting in the shard: all but the array's last run have >= minrun
  // keys, and merges with j in the shard are at most as many
  *h_cap = n_local / minrun_of(std::max<uint64_t>(n_total, 1)) + 2;
  return VMPS_OK;
}

static vmps_status_t merge_plan_dist_impl(vmps_comm_t c, const void* keys, uint64_t n_local, vmps_key_t kt,
                                          uint64_t* run_start, uint8_t* run_kind, vmps_merge_rec_t* merges,
                                          uint64_t cap_runs, uint64_t* h_num_runs_local,
                                          uint64_t* h_num_merges_local, void* ws, size_t ws_bytes, void* stream);

vmps_status_t vmps_merge_plan_dist(vmps_comm_t c, const void* keys, uint64_t n_local, vmps_key_t kt,
                                   uint64_t* run_start, uint8_t* run_kind, vmps_merge_rec_t* merges,
                                   uint64_t cap_runs, uint64_t* h_num_runs_local, uint64_t* h_num_merges_local,
                                   void* ws, size_t ws_bytes, void* stream) {
  return fail_group(c, merge_plan_dist_impl(c, keys, n_local, kt, run_start, run_kind, merges, cap_runs,
                                            h_num_runs_local, h_num_merges_local, ws, ws_bytes, stream));
}

static vmps_status_t merge_plan_dist_impl(vmps_comm_t c, const void* keys, uint64_t n_local, vmps_key_t kt,
                                          uint64_t* run_start, uint8_t* run_kind, vmps_merge_rec_t* merges,
                                          uint64_t cap_runs, uint64_t* h_num_runs_local,
                                          uint64_t* h_num_merges_local, void* ws, size_t ws_bytes, void* stream) {
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
  c_err.clear();
  std::vector<uint64_t> sizes;
  VK(gather_host(c, &n_local, 1, &sizes, d_small0, s));
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
  VK(tp_allgather(c, mine, d_edges, eb, s));
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
  VK(tp_allgather(c, tmine, d_tabs, (size_t)ns * 8, s));
  std::vector<uint64_t> tabs((size_t)g * ns);
  CK(cudaMemcpyAsync(tabs.data(), d_tabs, tabs.size() * 8, cudaMemcpyDeviceToHost, s));
  VK(tp_sync(c, s));
  std::vector<uint64_t> cnt(g, 0);
  std::vector<uint32_t> entry(g, 0);
  compose_tables((uint32_t)g, ns, tabs.data(), sizes.data(), entry.data(), cnt.data());
  std::vector<uint64_t> roff(g + 1, 0);
  for (int q = 0; q < g; ++q) roff[q + 1] = roff[q] + cnt[q];
  const uint64_t r = roff[g];
  if (r > rcap) { c_err = "internal: run capacity"; return VMPS_ERR_INTERNAL; }
  if (cnt[me])
    VK(vmps_shard_runs(keys, n_local, kt, mr, n_end, d_prev, nh ? d_halo : nullptr, nh, entry[me], cnt[me], off[me],
                       d_runs + roff[me], d_kinds + roff[me], shard_ws, std::max(L.shard_ws, L.plan_ws), s));
  // every rank's run list to every rank, in place, rank order
  {
    std::vector<BItem> items;
    for (int q = 0; q < g; ++q) {
      if (!cnt[q]) continue;
      items.push_back({d_runs + roff[q], cnt[q] * 8, q});
      items.push_back({d_kinds + roff[q], cnt[q], q});
    }
    VK(tp_bcast_many(c, items, s));
  }
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
    VK(tp_sync(c, s));
    if (nm > cap_runs) { c_err = "cap_runs too small for the merges"; *h_num_merges_local = nm; return VMPS_ERR_INVALID_ARG; }
    if (nm) {
      if (!merges) return VMPS_ERR_INVALID_ARG;
      CK(cudaMemcpyAsync(merges, d_recs, nm * sizeof(vmps_merge_rec_t), cudaMemcpyDeviceToDevice, s));
    }
  }
  *h_num_merges_local = nm;
  return tp_sync(c, s);
}

}  // extern "C"
