// NodeColumns halo exchange on the device (functionspace.py:58-118).
//
// Plan (functionspace.py:47-55): peers ascending; per peer the owned rows to send in the
// requester's order (functionspace.py:82-93), the ghost rows to receive in local
// (halo, gidx) order (functionspace.py:66-72), and each ghost's row on its owner
// (mesh.py:303-308, node_remote == the owner's send entry for it).
//
// Kernels (one warp per row, lanes over the row's items):
//   pack   — every peer's payload into one device buffer, peers ascending, (n, L) C-order:
//            byte-equal to f.host[send[peer]].tobytes() (functionspace.py:113-114)
//   unpack — receive buffer into the ghost rows (functionspace.py:115-117)
//   pull   — fused pack+transfer+unpack: each ghost row is read straight from its owner's
//            field through a peer pointer (same device, NVLink P2P, or a CUDA-IPC mapping).
// The NCCL path groups one ncclSend + ncclRecv per peer between pack and unpack on one
// stream.  NCCL is dlopen'ed on first use so the library never pins a libnccl version into
// a process that also loads torch's.
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <type_traits>
#include <vector>

#include "plan.cuh"

namespace sg {
namespace {

// Rows are moved as words of the field's item size (8 B for real64/int64, 4 B otherwise):
// W words per row, pitches in words.  Dense rows are item-aligned only, so no wider moves.
// A warp moves one row; every lane issues all its loads of the row before its stores
// (IT = ceil(W / 32) words per lane, 5 at 137 levels), so a row costs one memory latency —
// HBM, or NVLink for the peer reads of pull_rows — instead of one per 32-word slice.  Rows
// wider than 8 slices go in chunks of 4 slices.
template <typename Wd, int IT>
__device__ __forceinline__ void copy_row(Wd* __restrict__ dst, const Wd* __restrict__ src, int W, int lane) {
  if constexpr (IT > 0) {
    Wd v[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i)
      if (lane + 32 * i < W) v[i] = src[lane + 32 * i];
#pragma unroll
    for (int i = 0; i < IT; ++i)
      if (lane + 32 * i < W) dst[lane + 32 * i] = v[i];
  } else {
    for (int b = 0; b < W; b += 128) {
      Wd v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (b + lane + 32 * i < W) v[i] = src[b + lane + 32 * i];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (b + lane + 32 * i < W) dst[b + lane + 32 * i] = v[i];
    }
  }
}

template <typename Wd, int IT>
__global__ void __launch_bounds__(256) pack_rows(const Wd* __restrict__ f, int64_t pitch_w, int W,
                                                 const int32_t* __restrict__ rows, int64_t n, Wd* __restrict__ out) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  copy_row<Wd, IT>(out + r * W, f + (int64_t)rows[r] * pitch_w, W, threadIdx.x & 31);
}

template <typename Wd, int IT>
__global__ void __launch_bounds__(256) unpack_rows(Wd* __restrict__ f, int64_t pitch_w, int W,
                                                   const int32_t* __restrict__ rows, int64_t n,
                                                   const Wd* __restrict__ in) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  copy_row<Wd, IT>(f + (int64_t)rows[r] * pitch_w, in + r * W, W, threadIdx.x & 31);
}

struct PeerPtrs {
  const void* base[kMaxPeers];
  int64_t pitch_w[kMaxPeers];
};

// Fused exchange: ghost row k (peer slot s) <- the owner's row recv_remote[k], read through a
// peer pointer (same device, NVLink P2P or CUDA IPC): pack, transfer and unpack in one pass.
// A warp moves kPullRows rows, issuing the loads of all of them before any store (the copy is
// latency-bound with one row per warp: 4 x IT loads in flight per lane instead of IT).
constexpr int kPullRows = 4;

template <typename Wd, int IT>
__global__ void __launch_bounds__(256) pull_rows(Wd* __restrict__ f, int64_t pitch_w, int W,
                                                 const int32_t* __restrict__ rows, const int32_t* __restrict__ remote,
                                                 const int32_t* __restrict__ slot, int64_t n, PeerPtrs peers) {
  const int64_t r0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kPullRows;
  if (r0 >= n) return;
  const int lane = threadIdx.x & 31;
  if constexpr (IT == 0) {
    for (int64_t r = r0; r < min(r0 + kPullRows, n); ++r) {
      const int s = slot[r];
      const Wd* src = static_cast<const Wd*>(peers.base[s]) + (int64_t)remote[r] * peers.pitch_w[s];
      copy_row<Wd, 0>(f + (int64_t)rows[r] * pitch_w, src, W, lane);
    }
  } else {
    const Wd* src[kPullRows];
    Wd* dst[kPullRows];
#pragma unroll
    for (int q = 0; q < kPullRows; ++q) {
      const int64_t r = min(r0 + q, n - 1);  // a short tail repeats the last row (idempotent)
      const int s = slot[r];
      src[q] = static_cast<const Wd*>(peers.base[s]) + (int64_t)remote[r] * peers.pitch_w[s];
      dst[q] = f + (int64_t)rows[r] * pitch_w;
    }
    Wd v[kPullRows][IT];
#pragma unroll
    for (int q = 0; q < kPullRows; ++q)
#pragma unroll
      for (int i = 0; i < IT; ++i)
        if (lane + 32 * i < W) v[q][i] = src[q][lane + 32 * i];
#pragma unroll
    for (int q = 0; q < kPullRows; ++q)
#pragma unroll
      for (int i = 0; i < IT; ++i)
        if (lane + 32 * i < W) dst[q][lane + 32 * i] = v[q][i];
  }
}

// Launches KERNEL<Wd, IT> with IT = ceil(W / 32) (0 = chunked loop beyond 8 slices).
#define SG_ROW_KERNEL(KERNEL, Wd, W, GRID, STREAM, ...)                          \
  do {                                                                           \
    switch (((W) + 31) / 32) {                                                   \
      case 1: KERNEL<Wd, 1><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;       \
      case 2: KERNEL<Wd, 2><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;       \
      case 3: KERNEL<Wd, 3><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;       \
      case 4: KERNEL<Wd, 4><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;       \
      case 5: KERNEL<Wd, 5><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;       \
      case 6: KERNEL<Wd, 6><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;       \
      case 7: KERNEL<Wd, 7><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;       \
      case 8: KERNEL<Wd, 8><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;       \
      default: KERNEL<Wd, 0><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;      \
    }                                                                            \
  } while (0)

inline unsigned warps_grid(int64_t n) { return (unsigned)((n + 7) / 8); }

// ---- NCCL, loaded lazily --------------------------------------------------------------------
typedef int ncclResult_t;
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
  char internal[128];
};
enum { ncclUint8 = 1 };
struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommCuDevice)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};
std::mutex g_nccl_mu;
Nccl g_nccl;

Nccl& nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (!g_nccl.lib) {
    // SG_NCCL_LIBRARY (set by _native.py to the NCCL wheel torch links, when installed) first:
    // a process that later imports torch must find the same libnccl.so.2 already loaded —
    // an older system NCCL loaded under that soname breaks libtorch_cuda's symbol binding
    void* h = nullptr;
    if (const char* env = getenv("SG_NCCL_LIBRARY")) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw_error(SG_DOMAIN_ERROR, "NcclUnavailable: cannot dlopen libnccl.so.2: %s", dlerror());
#define SG_NCCL_SYM(field, name)                                                   \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));         \
  if (!g_nccl.field) throw_error(SG_DOMAIN_ERROR, "NcclUnavailable: missing %s", name);
    SG_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
    SG_NCCL_SYM(CommInitRank, "ncclCommInitRank");
    SG_NCCL_SYM(CommInitAll, "ncclCommInitAll");
    SG_NCCL_SYM(CommDestroy, "ncclCommDestroy");
    SG_NCCL_SYM(GroupStart, "ncclGroupStart");
    SG_NCCL_SYM(GroupEnd, "ncclGroupEnd");
    SG_NCCL_SYM(Send, "ncclSend");
    SG_NCCL_SYM(Recv, "ncclRecv");
    SG_NCCL_SYM(AllReduce, "ncclAllReduce");
    SG_NCCL_SYM(GetErrorString, "ncclGetErrorString");
    SG_NCCL_SYM(CommCount, "ncclCommCount");
    SG_NCCL_SYM(CommUserRank, "ncclCommUserRank");
    SG_NCCL_SYM(CommCuDevice, "ncclCommCuDevice");
    SG_NCCL_SYM(GetVersion, "ncclGetVersion");
#undef SG_NCCL_SYM
    g_nccl.lib = h;
  }
  return g_nccl;
}

#define SG_NCCL(call)                                                                         \
  do {                                                                                        \
    ncclResult_t _r = (call);                                                                 \
    if (_r != 0) throw_error(SG_DOMAIN_ERROR, "NcclError: %s failed: %s", #call,              \
                             nccl().GetErrorString(_r));                                      \
  } while (0)

struct Comm : Object {
  Comm() : Object(ObjKind::Comm) {}
  int device = 0, nranks = 0, rank = 0;
  ncclComm_t comm = nullptr;
  DevBuf token;  // 4-B device word for the stream-ordered barrier
  ~Comm() override {
    if (comm) nccl().CommDestroy(comm);
  }
};

// Dispatch on the field's item size: 8-byte kinds move as uint64, 4-byte kinds as uint32.
template <class F>
void by_word(const Field* f, F&& fn) {
  if (f->itemsize == 8) fn((uint64_t*)nullptr);
  else fn((uint32_t*)nullptr);
}

void check_field(const Plan* p, const Field* f) {
  if (f->npts != p->nnodes)
    throw_error(SG_DOMAIN_ERROR, "PlanMismatch: field has %lld points, plan covers %lld nodes",
                (long long)f->npts, (long long)p->nnodes);
  SG_REQUIRE(f->device == p->device, "field and plan live on different devices");
}

void upload_i32(DevBuf& b, int dev, const std::vector<int32_t>& v) {
  b.alloc(dev, std::max<size_t>(v.size(), 1) * 4);
  if (!v.empty()) SG_CUDA(cudaMemcpy(b.ptr, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
}

}  // namespace
}  // namespace sg

using namespace sg;

extern "C" {

int32_t sg_halo_plan_create(int32_t device, int64_t nnodes, int32_t npeers, const int32_t* peers,
                            const int64_t* send_counts, const int64_t* send_rows, const int64_t* recv_counts,
                            const int64_t* recv_rows, const int64_t* recv_remote_rows, uint64_t* out_plan) {
  SG_API_BEGIN
  SG_REQUIRE(out_plan, "null out pointer");
  SG_REQUIRE(npeers >= 0 && npeers <= kMaxPeers, "npeers %d outside [0, %d]", npeers, kMaxPeers);
  SG_REQUIRE(nnodes >= 0 && nnodes < INT32_MAX, "bad nnodes");
  auto p = std::make_unique<Plan>();
  p->device = device;
  p->nnodes = nnodes;
  p->send_off.assign(npeers + 1, 0);
  p->recv_off.assign(npeers + 1, 0);
  std::vector<int32_t> srows, rrows, rremote, rslot;
  for (int i = 0; i < npeers; ++i) {
    SG_REQUIRE(i == 0 || peers[i] > peers[i - 1], "peers must be strictly ascending");
    p->peers.push_back(peers[i]);
    p->send_off[i + 1] = p->send_off[i] + send_counts[i];
    p->recv_off[i + 1] = p->recv_off[i] + recv_counts[i];
  }
  const int64_t ns = p->send_off[npeers], nr = p->recv_off[npeers];
  for (int64_t k = 0; k < ns; ++k) {
    SG_REQUIRE(send_rows[k] >= 0 && send_rows[k] < nnodes, "send row %lld out of range", (long long)send_rows[k]);
    srows.push_back((int32_t)send_rows[k]);
  }
  p->has_remote = recv_remote_rows != nullptr;
  for (int i = 0; i < npeers; ++i)
    for (int64_t k = p->recv_off[i]; k < p->recv_off[i + 1]; ++k) {
      SG_REQUIRE(recv_rows[k] >= 0 && recv_rows[k] < nnodes, "recv row %lld out of range", (long long)recv_rows[k]);
      const int64_t rem = recv_remote_rows ? recv_remote_rows[k] : -1;
      // -1 = owner row unknown (a plan built from send/recv lists only); pack/unpack still work
      SG_REQUIRE(rem >= -1 && rem < INT32_MAX, "recv_remote row %lld out of range", (long long)rem);
      if (rem < 0) p->has_remote = false;
      rrows.push_back((int32_t)recv_rows[k]);
      rremote.push_back((int32_t)rem);
      rslot.push_back(i);
    }
  DeviceScope ds(device);
  upload_i32(p->send_rows, device, srows);
  upload_i32(p->recv_rows, device, rrows);
  upload_i32(p->recv_remote, device, rremote);
  upload_i32(p->recv_peer, device, rslot);
  // dense ghost map over [ghost_lo, nnodes): owner slot and owner row of every received row
  if (!rrows.empty()) {
    p->ghost_lo = *std::min_element(rrows.begin(), rrows.end());
    std::vector<int32_t> gs((size_t)(nnodes - p->ghost_lo), -1), gr((size_t)(nnodes - p->ghost_lo), -1);
    for (size_t k = 0; k < rrows.size(); ++k) {
      gs[rrows[k] - p->ghost_lo] = rslot[k];
      gr[rrows[k] - p->ghost_lo] = rremote[k];
    }
    upload_i32(p->ghost_slot, device, gs);
    upload_i32(p->ghost_row, device, gr);
  } else {
    p->ghost_lo = nnodes;
  }
  *out_plan = registry_put(p.release());
  SG_API_END
}

int32_t sg_halo_plan_info(uint64_t plan, int64_t* out_nsend, int64_t* out_nrecv) {
  SG_API_BEGIN
  Plan* p = get<Plan>(plan, ObjKind::Plan);
  if (out_nsend) *out_nsend = p->send_off.back();
  if (out_nrecv) *out_nrecv = p->recv_off.back();
  SG_API_END
}

int32_t sg_halo_pack(uint64_t plan, uint64_t field, void* dev_sendbuf, uint64_t stream) {
  SG_API_BEGIN
  Plan* p = get<Plan>(plan, ObjKind::Plan);
  Field* f = get<Field>(field, ObjKind::Field);
  check_field(p, f);
  const int64_t n = p->send_off.back();
  if (n == 0) return SG_OK;
  SG_REQUIRE(dev_sendbuf, "null send buffer");
  DeviceScope ds(p->device);
  by_word(f, [&](auto* tag) {
    using Wd = std::remove_pointer_t<decltype(tag)>;
    SG_ROW_KERNEL(pack_rows, Wd, f->levels, warps_grid(n), as_stream(stream), f->buf.as<Wd>(), f->pitch, f->levels,
                  p->send_rows.as<int32_t>(), n, static_cast<Wd*>(dev_sendbuf));
  });
  SG_CUDA_LAUNCH();
  SG_API_END
}

int32_t sg_halo_unpack(uint64_t plan, uint64_t field, const void* dev_recvbuf, uint64_t stream) {
  SG_API_BEGIN
  Plan* p = get<Plan>(plan, ObjKind::Plan);
  Field* f = get<Field>(field, ObjKind::Field);
  check_field(p, f);
  const int64_t n = p->recv_off.back();
  if (n == 0) return SG_OK;
  SG_REQUIRE(dev_recvbuf, "null receive buffer");
  DeviceScope ds(p->device);
  by_word(f, [&](auto* tag) {
    using Wd = std::remove_pointer_t<decltype(tag)>;
    SG_ROW_KERNEL(unpack_rows, Wd, f->levels, warps_grid(n), as_stream(stream), f->buf.as<Wd>(), f->pitch, f->levels,
                  p->recv_rows.as<int32_t>(), n, static_cast<const Wd*>(dev_recvbuf));
  });
  SG_CUDA_LAUNCH();
  SG_API_END
}

int32_t sg_halo_pull(uint64_t plan, uint64_t field, const uint64_t* peer_ptrs, const int64_t* peer_pitch_elems,
                     uint64_t stream) {
  SG_API_BEGIN
  Plan* p = get<Plan>(plan, ObjKind::Plan);
  Field* f = get<Field>(field, ObjKind::Field);
  check_field(p, f);
  const int64_t n = p->recv_off.back();
  if (n == 0) return SG_OK;
  SG_REQUIRE(peer_ptrs && peer_pitch_elems, "null peer arrays");
  SG_REQUIRE(p->has_remote, "plan has ghosts without an owner row (recv_remote); the pull transport needs them");
  PeerPtrs pp{};
  for (size_t i = 0; i < p->peers.size(); ++i) {
    pp.base[i] = reinterpret_cast<const void*>(peer_ptrs[i]);
    pp.pitch_w[i] = peer_pitch_elems[i];
    if (p->recv_off[i + 1] > p->recv_off[i]) SG_REQUIRE(pp.base[i], "null peer pointer for peer %d", p->peers[i]);
  }
  DeviceScope ds(p->device);
  by_word(f, [&](auto* tag) {
    using Wd = std::remove_pointer_t<decltype(tag)>;
    SG_ROW_KERNEL(pull_rows, Wd, f->levels, warps_grid((n + kPullRows - 1) / kPullRows), as_stream(stream),
                  f->buf.as<Wd>(), f->pitch, f->levels,
                  p->recv_rows.as<int32_t>(), p->recv_remote.as<int32_t>(), p->recv_peer.as<int32_t>(), n, pp);
  });
  SG_CUDA_LAUNCH();
  SG_API_END
}

int32_t sg_nccl_unique_id(uint8_t* out_id, size_t n) {
  SG_API_BEGIN
  SG_REQUIRE(out_id && n >= sizeof(ncclUniqueId), "buffer must hold %zu bytes", sizeof(ncclUniqueId));
  ncclUniqueId id;
  SG_NCCL(nccl().GetUniqueId(&id));
  memcpy(out_id, &id, sizeof(id));
  SG_API_END
}

int32_t sg_comm_create(int32_t device, int32_t nranks, int32_t rank, const uint8_t* id, size_t n,
                       uint64_t* out_comm) {
  SG_API_BEGIN
  SG_REQUIRE(out_comm && id && n >= sizeof(ncclUniqueId), "bad arguments");
  SG_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "rank %d not in [0, %d)", rank, nranks);
  DeviceScope ds(device);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  auto c = std::make_unique<Comm>();
  c->device = device;
  c->nranks = nranks;
  c->rank = rank;
  SG_NCCL(nccl().CommInitRank(&c->comm, nranks, uid, rank));
  c->token.alloc(device, 16);  // barrier word: allocated here, never inside a graph capture
  SG_CUDA(cudaMemset(c->token.ptr, 0, 16));
  *out_comm = registry_put(c.release());
  SG_API_END
}

// One process driving several GPUs (in-process ranks, one host thread per GPU): one
// communicator per device from ncclCommInitAll; rank r of the set runs on devices[r].
int32_t sg_comm_init_all(int32_t ndev, const int32_t* devices, uint64_t* out_comms) {
  SG_API_BEGIN
  SG_REQUIRE(ndev >= 1 && devices && out_comms, "bad arguments");
  std::vector<ncclComm_t> comms((size_t)ndev, nullptr);
  std::vector<int> devs(devices, devices + ndev);
  SG_NCCL(nccl().CommInitAll(comms.data(), ndev, devs.data()));
  for (int r = 0; r < ndev; ++r) {
    DeviceScope ds(devs[(size_t)r]);
    auto c = std::make_unique<Comm>();
    c->device = devs[(size_t)r];
    c->nranks = ndev;
    c->rank = r;
    c->comm = comms[(size_t)r];
    comms[(size_t)r] = nullptr;
    c->token.alloc(c->device, 16);
    SG_CUDA(cudaMemset(c->token.ptr, 0, 16));
    out_comms[r] = registry_put(c.release());
  }
  SG_API_END
}

// NCCL's own view of a communicator (ncclCommCount / ncclCommUserRank / ncclCommCuDevice)
// and the loaded library's version code: evidence that a multi-rank run really used NCCL.
int32_t sg_comm_info(uint64_t comm, int32_t* out_nranks, int32_t* out_rank, int32_t* out_device,
                     int32_t* out_version) {
  SG_API_BEGIN
  Comm* c = get<Comm>(comm, ObjKind::Comm);
  Nccl& N = nccl();
  int v = 0;
  if (out_nranks) {
    SG_NCCL(N.CommCount(c->comm, &v));
    *out_nranks = v;
  }
  if (out_rank) {
    SG_NCCL(N.CommUserRank(c->comm, &v));
    *out_rank = v;
  }
  if (out_device) {
    SG_NCCL(N.CommCuDevice(c->comm, &v));
    *out_device = v;
  }
  if (out_version) {
    SG_NCCL(N.GetVersion(&v));
    *out_version = v;
  }
  SG_API_END
}

// Stream-ordered barrier: an ncclAllReduce of one word on `stream`.  Work enqueued after it
// on any rank starts only once every rank's earlier work on its stream has completed — the
// fence the fused exchange+apply needs around peer reads, without a host round trip, and
// capturable into a CUDA graph.
int32_t sg_comm_barrier(uint64_t comm, uint64_t stream) {
  SG_API_BEGIN
  Comm* c = get<Comm>(comm, ObjKind::Comm);
  DeviceScope ds(c->device);
  SG_NCCL(nccl().AllReduce(c->token.ptr, c->token.ptr, 1, /*ncclInt32*/ 2, /*ncclSum*/ 0, c->comm, as_stream(stream)));
  SG_API_END
}

int32_t sg_halo_exchange_nccl(uint64_t plan, uint64_t field, uint64_t comm, uint64_t stream) {
  SG_API_BEGIN
  Plan* p = get<Plan>(plan, ObjKind::Plan);
  Field* f = get<Field>(field, ObjKind::Field);
  Comm* c = get<Comm>(comm, ObjKind::Comm);
  check_field(p, f);
  DeviceScope ds(p->device);
  cudaStream_t st = as_stream(stream);
  const int64_t ns = p->send_off.back(), nr = p->recv_off.back();
  const size_t row = (size_t)f->levels * f->itemsize;  // payload bytes per row
  if ((size_t)ns * row > p->sendbuf.bytes) p->sendbuf.alloc(p->device, (size_t)ns * row);
  if ((size_t)nr * row > p->recvbuf.bytes) p->recvbuf.alloc(p->device, (size_t)nr * row);
  if (ns) {
    by_word(f, [&](auto* tag) {
      using Wd = std::remove_pointer_t<decltype(tag)>;
      SG_ROW_KERNEL(pack_rows, Wd, f->levels, warps_grid(ns), st, f->buf.as<Wd>(), f->pitch, f->levels,
                    p->send_rows.as<int32_t>(), ns, p->sendbuf.as<Wd>());
    });
    SG_CUDA_LAUNCH();
  }
  Nccl& N = nccl();
  SG_NCCL(N.GroupStart());
  for (size_t i = 0; i < p->peers.size(); ++i) {
    const int64_t s0 = p->send_off[i], s1 = p->send_off[i + 1];
    const int64_t r0 = p->recv_off[i], r1 = p->recv_off[i + 1];
    if (s1 > s0) SG_NCCL(N.Send(p->sendbuf.as<char>() + s0 * row, (size_t)(s1 - s0) * row, ncclUint8, p->peers[i], c->comm, st));
    if (r1 > r0) SG_NCCL(N.Recv(p->recvbuf.as<char>() + r0 * row, (size_t)(r1 - r0) * row, ncclUint8, p->peers[i], c->comm, st));
  }
  SG_NCCL(N.GroupEnd());
  if (nr) {
    by_word(f, [&](auto* tag) {
      using Wd = std::remove_pointer_t<decltype(tag)>;
      SG_ROW_KERNEL(unpack_rows, Wd, f->levels, warps_grid(nr), st, f->buf.as<Wd>(), f->pitch, f->levels,
                    p->recv_rows.as<int32_t>(), nr, p->recvbuf.as<Wd>());
    });
    SG_CUDA_LAUNCH();
  }
  SG_API_END
}

int32_t sg_ipc_handle(uint64_t field, uint8_t* out_handle, size_t n) {
  SG_API_BEGIN
  Field* f = get<Field>(field, ObjKind::Field);
  SG_REQUIRE(out_handle && n >= sizeof(cudaIpcMemHandle_t), "buffer must hold %zu bytes", sizeof(cudaIpcMemHandle_t));
  DeviceScope ds(f->device);
  cudaIpcMemHandle_t h;
  SG_CUDA(cudaIpcGetMemHandle(&h, f->buf.ptr));
  memcpy(out_handle, &h, sizeof(h));
  SG_API_END
}

int32_t sg_ipc_open(int32_t device, const uint8_t* handle, size_t n, uint64_t* out_ptr) {
  SG_API_BEGIN
  SG_REQUIRE(handle && out_ptr && n >= sizeof(cudaIpcMemHandle_t), "bad arguments");
  DeviceScope ds(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* ptr = nullptr;
  SG_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
  *out_ptr = reinterpret_cast<uint64_t>(ptr);
  SG_API_END
}

int32_t sg_ipc_close(int32_t device, uint64_t ptr) {
  SG_API_BEGIN
  DeviceScope ds(device);
  SG_CUDA(cudaIpcCloseMemHandle(reinterpret_cast<void*>(ptr)));
  SG_API_END
}

}  // extern "C"
