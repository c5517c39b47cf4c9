// One distributed remap step as ONE kernel per rank: halo exchange over peer memory + apply,
// fenced by device-side signals instead of host or NCCL barriers; and the halo exchange alone
// as one signalled pull kernel per rank (cfg4).
//
// The reference step of a partition is halo_exchange (functionspace.py:107-118: owners'
// values land in the ghost rows) followed by apply_remap (interp.py:206-228), in that order
// (cli.py:138-144).  Here the two fuse (as in fused.cu: boundary targets read their ghost
// stencil rows straight from the owners' HBM through peer pointers, NVLink P2P or CUDA IPC),
// and the two barriers around the peer reads become flag words in device memory:
//
//   signal kernel (one thread per rank):
//       e = epoch + 1;  for every rank that reads my rows: st.release  its ready[me] = e;
//       then (all ranks of the launch published) ld.acquire  ready[owner] >= e  for every owner
//   step kernel (targets in natural order, one warp each; launched with PDL, so it starts
//   while the signal kernel still waits):
//       interior targets (every stencil row owned): apply from local rows — no wait;
//       boundary targets: griddepcontrol.wait (the signal kernel saw every owner's ready
//         word), then apply with the ghost rows read from the owners' fields; each counts
//         itself (acq_rel atomic) and the last one st.release-es done[me] = e to every owner
//         and, with one GPU per rank, waits for done[reader] >= e from every reader of my
//         rows — after that nobody reads my rows any more, so the caller may overwrite them;
//         epoch = e.
// Flag accesses use the peer's scope: .sys for a peer on another GPU, .gpu for a rank on the
// same GPU (a .sys release under load costs tens of µs, profiles/r02_exchange_signalled.md).
//
// Both waits depend only on the OTHER ranks' signal kernels (which publish before they wait)
// and boundary warps, never on a block of the same launch, so with one GPU per rank there is no
// cycle.  Several ranks on ONE GPU
// must not run as separate launches that wait on each other (B200_PROFILING.md): for that case
// sg_step_launch takes every rank's step in ONE launch (block ranges per rank); the ready flags
// were then set by the preceding signal kernel, and the tail wait is left to the host
// (wait_done = 0; sg_signal_read checks the words).  Waits are bounded (10 s by default): on
// timeout the error word is set and the kernel continues; sg_step_check reports it (no hang,
// no silent result).
//
// Arithmetic identical to the apply kernels: bitwise equal to interp.py:219-223.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "plan.cuh"
#include "stencil.cuh"

namespace sg {

// Signal words (uint64) of one rank, zeroed at creation.
// Signal words allocated by THIS process, by address -> device.  A peer's words found here are
// a same-process rank (the single-GPU emulation, or in-process ranks on other GPUs); anything
// else (CUDA-IPC mappings of another process's words) is treated as another GPU: system scope.
std::mutex g_local_signals_mu;
std::unordered_map<uintptr_t, int> g_local_signals;

struct Signal : Object {
  Signal() : Object(ObjKind::Signal) {}
  ~Signal() override {
    std::lock_guard<std::mutex> lk(g_local_signals_mu);
    g_local_signals.erase(reinterpret_cast<uintptr_t>(words.ptr));
  }
  int device = 0;
  int32_t nranks = 0, rank = 0;
  DevBuf words;
  size_t nwords() const { return 2 * (size_t)nranks + 4; }
};

namespace {

constexpr int kMaxGroup = 16;  // ranks in one launch (single-GPU emulation)
constexpr int kRoleRecv = 1;   // I read this peer's rows (it owns some of my ghosts)
constexpr int kRoleSend = 2;   // this peer reads my rows
constexpr unsigned long long kTimeoutNs = 10ull * 1000 * 1000 * 1000;  // default wait bound

// word offsets
__host__ __device__ inline int w_ready(int r) { return r; }
__host__ __device__ inline int w_done(int nr, int r) { return nr + r; }
__host__ __device__ inline int w_epoch(int nr) { return 2 * nr; }
__host__ __device__ inline int w_cur(int nr) { return 2 * nr + 1; }
__host__ __device__ inline int w_count(int nr) { return 2 * nr + 2; }
__host__ __device__ inline int w_error(int nr) { return 2 * nr + 3; }

// Peers of one rank, BY VALUE in the kernel parameters (constant bank): the signal words,
// field pointers and roles of at most kPeers neighbours — no dependent global load on the
// signalling path or in front of a peer-row load.
constexpr int kPeers = 16;
struct PeerTable {
  int32_t npeers;
  int32_t rank[kPeers];
  unsigned char role[kPeers];
  unsigned char sys[kPeers];  // the peer is another GPU: flag accesses at system scope
  const void* base_any[kPeers];
  int64_t pitch[kPeers];  // elements
  unsigned long long* flags[kPeers];
};

// Everything a target warp needs, passed BY VALUE in the kernel parameters (constant bank):
// a warp reaches its stencil load with no dependent global load in front of it.
struct StepArgs {
  const int4* idx;
  const double2* w;  // double4 as two double2
  int64_t m;           // targets, processed in their natural (ascending) order
  int64_t n_boundary;  // targets with a ghost stencil row
  int32_t levels, k;
  const double* src;
  int64_t src_pitch;
  double* dst;
  int64_t dst_pitch;
  int64_t ghost_lo;  // local rows >= ghost_lo are ghosts: read from their owners
  const int32_t* ghost_slot;
  const int32_t* ghost_row;
  unsigned long long* flags;  // this rank's words
  unsigned long long timeout_ns;
  int32_t nranks, rank;
  PeerTable peers;
};

struct Group {
  StepArgs d[kMaxGroup];
  int64_t start[kMaxGroup + 1];  // first block of each rank
  int32_t n;
  int32_t wait_done;
};
static_assert(sizeof(Group) <= 32000, "kernel parameters are limited to 32764 bytes");

// Scope of a flag access: .sys when the other side of the flag is another GPU (NVLink / IPC),
// .gpu when it is this GPU (ranks of a single-GPU emulation) — a .sys release under load costs
// tens of µs more than a .gpu one (tools/xchg_sweep.py, profiles/r02_fused_step.md).
// One fence + relaxed (strong) accesses instead of a release / acquire per peer: a release
// fence followed by a strong store is a release pattern, a strong load followed by an acquire
// fence an acquire pattern (PTX memory model) — one MEMBAR per rank instead of one per peer.
__device__ __forceinline__ void fence_acq_rel(bool sys) {
  if (sys)
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  else
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p, bool sys) {
  unsigned long long v;
  if (sys)
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v, bool sys) {
  if (sys)
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Programmatic dependent launch: the signal kernel lets the step / pull kernel start at once
// (interior targets need nothing from it); code that reads the current epoch the signal kernel
// wrote first waits for the signal grid (griddepcontrol.wait = full completion + visibility).
__device__ __forceinline__ void pdl_release_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait_primary() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// acq_rel RMW at gpu scope: orders this block's peer reads (made visible to thread 0 by the
// preceding __syncthreads) before the count the finisher acquires.
__device__ __forceinline__ unsigned long long atom_add_acq_rel(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

// Spin until *p >= e (strong relaxed loads: the caller fences once after all its waits);
// false (and the error word set) after timeout_ns.
__device__ bool wait_geq(const unsigned long long* p, unsigned long long e, unsigned long long* err, int code,
                         unsigned long long timeout_ns, bool sys) {
  if (ld_relaxed(p, sys) >= e) return true;
  const unsigned long long t0 = now_ns();
  while (ld_relaxed(p, sys) < e) {
    __nanosleep(64);
    if (now_ns() - t0 > timeout_ns) {
      atomicExch(err, (unsigned long long)code);
      return false;
    }
  }
  return true;
}

__device__ __forceinline__ double ld_local(const double* p) {  // read-only for this launch
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_any(const double* p) {  // peer rows: written before the acquire
  double v;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_weak(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_weak(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double combine(double w0, double w1, double w2, double x, double y, double z) {
  return __dadd_rn(__dadd_rn(__dmul_rn(w0, x), __dmul_rn(w1, y)), __dmul_rn(w2, z));
}

__device__ __forceinline__ const double* row_of(const StepArgs& d, int n) {
  if (n < d.ghost_lo) return d.src + (int64_t)n * d.src_pitch;
  const int g = n - (int)d.ghost_lo;
  const int s = __ldg(d.ghost_slot + g);
  return static_cast<const double*>(d.peers.base_any[s]) + (int64_t)__ldg(d.ghost_row + g) * d.peers.pitch[s];
}

// One target per warp.  BOUNDARY: rows may live on peers (weak loads after the acquire).
template <int ITERS, bool BOUNDARY>
__device__ __forceinline__ void apply_target(const StepArgs& d, int64_t t, int4 id, int lane) {
  const double2 wa = __ldg(d.w + 2 * t), wb = __ldg(d.w + 2 * t + 1);
  const double *r0, *r1, *r2, *r3;
  if (BOUNDARY) {
    r0 = row_of(d, id.x);
    r1 = row_of(d, id.y);
    r2 = row_of(d, id.z);
    r3 = d.k == 4 ? row_of(d, id.w) : r0;
  } else {
    r0 = d.src + (int64_t)id.x * d.src_pitch;
    r1 = d.src + (int64_t)id.y * d.src_pitch;
    r2 = d.src + (int64_t)id.z * d.src_pitch;
    r3 = d.k == 4 ? d.src + (int64_t)id.w * d.src_pitch : r0;
  }
  double* out = d.dst + t * d.dst_pitch;
  const int L = d.levels;
  if (ITERS > 0) {
    double v0[ITERS > 0 ? ITERS : 1], v1[ITERS > 0 ? ITERS : 1], v2[ITERS > 0 ? ITERS : 1],
        v3[ITERS > 0 ? ITERS : 1];
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const int l = lane + 32 * i;
      if (l < L) {
        v0[i] = BOUNDARY ? ld_any(r0 + l) : ld_local(r0 + l);
        v1[i] = BOUNDARY ? ld_any(r1 + l) : ld_local(r1 + l);
        v2[i] = BOUNDARY ? ld_any(r2 + l) : ld_local(r2 + l);
        v3[i] = d.k == 4 ? (BOUNDARY ? ld_any(r3 + l) : ld_local(r3 + l)) : 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const int l = lane + 32 * i;
      if (l < L) {
        double o = combine(wa.x, wa.y, wb.x, v0[i], v1[i], v2[i]);
        if (d.k == 4) o = __dadd_rn(o, __dmul_rn(wb.y, v3[i]));
        __stcs(out + l, o);
      }
    }
  } else {
    for (int l = lane; l < L; l += 32) {
      double o = BOUNDARY ? combine(wa.x, wa.y, wb.x, ld_any(r0 + l), ld_any(r1 + l), ld_any(r2 + l))
                          : combine(wa.x, wa.y, wb.x, ld_local(r0 + l), ld_local(r1 + l), ld_local(r2 + l));
      if (d.k == 4) o = __dadd_rn(o, __dmul_rn(wb.y, BOUNDARY ? ld_any(r3 + l) : ld_local(r3 + l)));
      __stcs(out + l, o);
    }
  }
}


// The rank's last act of a step (one thread): tell the owners I am done reading their rows,
// then (one GPU per rank) wait until every reader of my rows is done; epoch = e.
__device__ void finish_epoch(unsigned long long* f, int nr, int rank, const PeerTable& P, unsigned long long e,
                             int wait_done, unsigned long long timeout_ns) {
  // one release fence orders this thread's (and, through the acq_rel count, every counted
  // block's) earlier reads of the peers' rows before every done word
  bool any = false, sys = false;
  for (int s = 0; s < P.npeers; ++s)
    if (P.role[s] & kRoleRecv) any = true, sys |= P.sys[s];
  if (any) fence_acq_rel(sys);
  for (int s = 0; s < P.npeers; ++s)
    if (P.role[s] & kRoleRecv) st_relaxed(P.flags[s] + w_done(nr, rank), e, P.sys[s]);
  if (wait_done) {
    bool wsys = false, waited = false;
    for (int s = 0; s < P.npeers; ++s)
      if (P.role[s] & kRoleSend) {
        wait_geq(f + w_done(nr, P.rank[s]), e, f + w_error(nr), 2, timeout_ns, P.sys[s]);
        waited = true, wsys |= P.sys[s];
      }
    if (waited) fence_acq_rel(wsys);  // acquire: the readers are done before the next epoch writes
  }
  f[w_count(nr)] = 0;
  f[w_epoch(nr)] = e;
}
__device__ void finish_step(const StepArgs& d, unsigned long long e, int wait_done) {
  finish_epoch(d.flags, d.nranks, d.rank, d.peers, e, wait_done, d.timeout_ns);
}
// The signal kernels: one thread per (rank, peer slot) of the launch, so the flag accesses of
// all peers go out in parallel instead of one after another.
//  * publish: ready[me] = epoch + 1 into every reader's words.  The owned rows were written by
//    earlier kernels of this stream (complete); a release fence + strong store orders them
//    before the ready word at the reader's scope (no separate fence.sc.sys: 18 µs here).
//  * after __syncthreads (every rank of a single-GPU emulation has published): wait until each
//    owner of this rank's ghosts published the same epoch, then an acquire fence.  The step /
//    pull kernel that depends on the signal kernel (griddepcontrol.wait) reads the owners' rows
//    without an acquire of its own.
constexpr int kSignalThreads = kMaxGroup * kPeers;

template <class G>
__device__ void signal_body(const G& g, bool (*needs_owners)(const G&, int)) {
  const int r = threadIdx.x / kPeers, s = threadIdx.x % kPeers;
  const bool rank_ok = r < g.n;
  const bool live = rank_ok && s < g.d[r].peers.npeers;
  unsigned long long* f = rank_ok ? g.d[r].flags : nullptr;
  const int nr = rank_ok ? g.d[r].nranks : 0;
  const unsigned long long e = rank_ok ? f[w_epoch(nr)] + 1 : 0;
  if (rank_ok && s == 0) f[w_cur(nr)] = e;
  if (live && (g.d[r].peers.role[s] & kRoleSend)) {
    const bool sys = g.d[r].peers.sys[s];
    fence_acq_rel(sys);
    st_relaxed(g.d[r].peers.flags[s] + w_ready(g.d[r].rank), e, sys);
  }
  __syncthreads();
  if (live && (g.d[r].peers.role[s] & kRoleRecv) && needs_owners(g, r)) {
    const bool sys = g.d[r].peers.sys[s];
    wait_geq(f + w_ready(g.d[r].peers.rank[s]), e, f + w_error(nr), 1, g.d[r].timeout_ns, sys);
    fence_acq_rel(sys);  // acquire pattern over the owner's ready word
  }
}

__device__ bool step_needs_owners(const Group& g, int r) { return g.d[r].n_boundary > 0; }

__global__ void __launch_bounds__(kSignalThreads) signal_kernel(Group g) {
  // launched with PDL too: it may start during the previous kernel's last wave (which calls
  // launch_dependents), but waits for that kernel's completion and memory before it reads the
  // epoch or publishes anything — only its launch latency is hidden
  pdl_wait_primary();
  pdl_release_dependents();
  signal_body(g, step_needs_owners);
}

constexpr int kWarps = 2;  // targets per block: small blocks retire and refill (apply.cu)

// Targets in natural order, one per warp.  A warp whose stencil touches a ghost row waits for
// the owners' ready words, reads the ghost rows from the owners' fields, and counts itself;
// the last such warp (or, with no boundary targets, warp 0 of block 0) finishes the step.
template <int ITERS>
__global__ void __launch_bounds__(kWarps * 32) step_kernel(Group g) {
  pdl_release_dependents();  // the next signal kernel may launch during the last wave
  int r = 0;
  while (r + 1 < g.n && (int64_t)blockIdx.x >= g.start[r + 1]) ++r;
  const StepArgs& d = g.d[r];
  const int64_t b = (int64_t)blockIdx.x - g.start[r];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = b * kWarps + warp;
  if (t >= d.m) {
    if (d.m == 0 && t == 0 && lane == 0) {  // no targets: still tell the owners, wait for readers
      pdl_wait_primary();
      finish_step(d, *(volatile unsigned long long*)(d.flags + w_cur(d.nranks)), g.wait_done);
    }
    return;
  }
  const int4 id = __ldg(d.idx + t);
  const int hi = max(max(id.x, id.y), d.k == 4 ? max(id.z, id.w) : id.z);
  if (hi < d.ghost_lo) {  // interior: local rows only, no wait
    apply_target<ITERS, false>(d, t, id, lane);
    if (d.n_boundary == 0 && t == 0 && lane == 0) {
      pdl_wait_primary();
      finish_step(d, *(volatile unsigned long long*)(d.flags + w_cur(d.nranks)), g.wait_done);
    }
    return;
  }
  unsigned long long* f = d.flags;
  const int nr = d.nranks;
  pdl_wait_primary();  // the signal kernel has seen every owner's ready word for this epoch
  const unsigned long long e = *(volatile unsigned long long*)(f + w_cur(nr));
  apply_target<ITERS, true>(d, t, id, lane);
  __syncwarp();
  if (lane == 0 && (int64_t)atom_add_acq_rel(f + w_count(nr), 1ull) == d.n_boundary - 1)
    finish_step(d, e, g.wait_done);  // all peer reads done
}

__global__ void count_boundary(const int4* idx, int64_t m, int k, int64_t ghost_lo, unsigned long long* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool bnd = false;
  if (t < m) {
    const int4 id = idx[t];
    const int hi = max(max(id.x, id.y), k == 4 ? max(id.z, id.w) : id.z);
    bnd = hi >= ghost_lo;
  }
  const unsigned c = __popc(__ballot_sync(0xffffffffu, bnd));
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// ---- the halo exchange alone, signalled (cfg4): ghost rows pulled from their owners ----
// functionspace.py:107-118 as one kernel per rank: warp per ghost row, waits for the owner's
// ready word, copies the owner's row (recv_remote) through the peer pointer into the ghost
// row; the last row's warp publishes done to the owners and waits for its own readers.
struct XchgArgs {
  void* base;
  int64_t pitch;  // elements (= words of the item size)
  int32_t W;      // words per row (levels)
  const int32_t* rows;    // ghost rows (local)
  const int32_t* remote;  // owner row of each ghost
  const int32_t* slot;    // owner's plan peer slot of each ghost
  int64_t n;
  unsigned long long* flags;
  unsigned long long timeout_ns;
  int32_t nranks, rank;
  PeerTable peers;
};

struct XGroup {
  XchgArgs d[kMaxGroup];
  int64_t start[kMaxGroup + 1];
  int32_t n;
  int32_t wait_done;
};
static_assert(sizeof(XGroup) <= 32000, "kernel parameters are limited to 32764 bytes");

constexpr int kXWarps = 8;

__device__ bool xchg_needs_owners(const XGroup& g, int r) { return g.d[r].n > 0; }

__global__ void __launch_bounds__(kSignalThreads) xsignal_kernel(XGroup g) {
  pdl_wait_primary();  // as signal_kernel
  pdl_release_dependents();
  signal_body(g, xchg_needs_owners);
}

// A block moves kXRows ghost rows per warp (kXWarps warps): after griddepcontrol.wait (the
// signal kernel saw every owner's ready word) every warp issues the loads of all its rows
// before its stores (4 rows x IT words in flight per lane: the copy is latency-bound
// otherwise); the last block to finish (acq_rel count) finishes the epoch.
constexpr int kXRows = 4;
constexpr int kXBlocksPerSM = 3;  // 256 threads x 80 registers: 3 resident blocks per SM (r02_exchange_xblocks.jsonl)

template <typename Wd, int IT>
__global__ void __launch_bounds__(kXWarps * 32) xchg_kernel(XGroup g) {
  pdl_release_dependents();  // the next signal kernel may launch during the last wave
  int r = 0;
  while (r + 1 < g.n && (int64_t)blockIdx.x >= g.start[r + 1]) ++r;
  const XchgArgs& d = g.d[r];
  const int64_t b = (int64_t)blockIdx.x - g.start[r], nb = g.start[r + 1] - g.start[r];
  const int lane = threadIdx.x & 31;
  unsigned long long* f = d.flags;
  const int nr = d.nranks;
  const PeerTable& P = d.peers;
  // resident grid: each warp moves kXRows rows per iteration, blocks stride over the rank's rows
  const int64_t stride = nb * kXWarps * kXRows;
  int64_t i0 = (b * kXWarps + (threadIdx.x >> 5)) * kXRows;
  // the next iteration's ghost / owner / slot indices are loaded while this iteration's rows
  // are in flight: one memory round trip per iteration instead of two
  int nslot[kXRows], nrem[kXRows], nrow[kXRows];
  if (IT > 0 && i0 < d.n) {
#pragma unroll
    for (int q = 0; q < kXRows; ++q) {
      const int64_t i = min(i0 + q, d.n - 1);  // a short tail repeats the last row (idempotent)
      nslot[q] = __ldg(d.slot + i);
      nrem[q] = __ldg(d.remote + i);
      nrow[q] = __ldg(d.rows + i);
    }
  }
  // (the plan's index arrays are static: their first loads above overlap the signal kernel)
  pdl_wait_primary();  // the signal kernel has seen every owner's ready word for this epoch
  const unsigned long long e_sh = *(volatile unsigned long long*)(f + w_cur(nr));
  for (; i0 < d.n; i0 += stride) {
    if (IT > 0) {
      const Wd* src[kXRows];
      Wd* dst[kXRows];
#pragma unroll
      for (int q = 0; q < kXRows; ++q) {
        const int s = nslot[q];
        src[q] = static_cast<const Wd*>(P.base_any[s]) + (int64_t)nrem[q] * P.pitch[s];
        dst[q] = static_cast<Wd*>(d.base) + (int64_t)nrow[q] * d.pitch;
      }
      Wd v[kXRows][IT > 0 ? IT : 1];
#pragma unroll
      for (int q = 0; q < kXRows; ++q)
#pragma unroll
        for (int k = 0; k < IT; ++k)
          if (lane + 32 * k < d.W) v[q][k] = ld_weak(src[q] + lane + 32 * k);
      if (i0 + stride < d.n) {
#pragma unroll
        for (int q = 0; q < kXRows; ++q) {
          const int64_t i = min(i0 + stride + q, d.n - 1);
          nslot[q] = __ldg(d.slot + i);
          nrem[q] = __ldg(d.remote + i);
          nrow[q] = __ldg(d.rows + i);
        }
      }
#pragma unroll
      for (int q = 0; q < kXRows; ++q)
#pragma unroll
        for (int k = 0; k < IT; ++k)
          if (lane + 32 * k < d.W) dst[q][lane + 32 * k] = v[q][k];
    } else {
      for (int64_t i = i0; i < min(i0 + kXRows, d.n); ++i) {
        const int s = __ldg(d.slot + i);
        const Wd* src = static_cast<const Wd*>(P.base_any[s]) + (int64_t)__ldg(d.remote + i) * P.pitch[s];
        Wd* dst = static_cast<Wd*>(d.base) + (int64_t)__ldg(d.rows + i) * d.pitch;
        for (int k = lane; k < d.W; k += 32) dst[k] = ld_weak(src + k);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && atom_add_acq_rel(f + w_count(nr), 1ull) == (unsigned long long)(nb - 1))
    finish_epoch(f, nr, d.rank, P, e_sh, g.wait_done, d.timeout_ns);  // all reads of peers' rows done
}

// Launch with programmatic stream serialization: may start while the preceding kernel of the
// stream (the signal kernel) is still running; the kernel calls pdl_wait_primary() where needed.
// cooperative = true instead: every block co-resident (checked), no PDL — the single-GPU
// emulation in which the ranks' tail waits (wait_done) may spin on each other's blocks.
template <class G>
void launch_pdl(void (*kernel)(G), unsigned grid, unsigned block, cudaStream_t s, const G& g,
                bool cooperative = false) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (cooperative) {
    int dev = 0, nsm = 0, per_sm = 0;
    SG_CUDA(cudaGetDevice(&dev));
    SG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, (int)block, 0));
    SG_REQUIRE((int64_t)grid <= (int64_t)per_sm * nsm,
               "cooperative launch of %u blocks exceeds the %d x %d co-resident blocks", grid, per_sm, nsm);
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  } else {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SG_CUDA(cudaLaunchKernelEx(&cfg, kernel, g));
}

struct Exchange : Object {
  Exchange() : Object(ObjKind::Exchange) {}
  int device = 0;
  int itemsize = 8;
  XchgArgs args{};
  uint64_t signal = 0;
};

struct Step : Object {
  Step() : Object(ObjKind::Step) {}
  int device = 0;
  StepArgs args{};
  int64_t nblocks = 0;
  uint64_t signal = 0;
};

// Peers of a plan for a signalled launch: role bits from the plan's send / recv lists, the
// owners' field pointers (needed where this rank receives) and every peer's signal words.
PeerTable peer_table(const Plan* p, const Signal* sig, const uint64_t* peer_ptrs, const int64_t* peer_pitch_elems,
                     const uint64_t* peer_flag_ptrs) {
  const size_t np = p->peers.size();
  SG_REQUIRE(np <= (size_t)kPeers, "%zu peers: signalled launches take at most %d", np, kPeers);
  SG_REQUIRE(np == 0 || (peer_ptrs && peer_pitch_elems && peer_flag_ptrs), "null peer arrays");
  SG_REQUIRE(p->recv_off.back() == 0 || p->has_remote,
             "plan has ghosts without an owner row (recv_remote); signalled peer reads need them");
  PeerTable pt{};
  pt.npeers = (int32_t)np;
  for (size_t i = 0; i < np; ++i) {
    SG_REQUIRE(p->peers[i] >= 0 && p->peers[i] < sig->nranks && p->peers[i] != sig->rank,
               "plan peer %d is not another rank of %d", p->peers[i], sig->nranks);
    SG_REQUIRE(peer_flag_ptrs[i] != 0, "null signal words for peer %d", p->peers[i]);
    pt.rank[i] = p->peers[i];
    pt.role[i] = (p->recv_off[i + 1] > p->recv_off[i] ? kRoleRecv : 0) |
                 (p->send_off[i + 1] > p->send_off[i] ? kRoleSend : 0);
    SG_REQUIRE(!(pt.role[i] & kRoleRecv) || peer_ptrs[i] != 0, "null field pointer for peer %d", p->peers[i]);
    pt.base_any[i] = reinterpret_cast<const void*>(peer_ptrs[i]);
    pt.pitch[i] = peer_pitch_elems[i];
    pt.flags[i] = reinterpret_cast<unsigned long long*>(peer_flag_ptrs[i]);
    // .gpu scope only for a peer whose signal words this process allocated on this very device
    // (ranks of a single-GPU emulation); IPC mappings and other GPUs: .sys
    int peer_dev = -1;
    {
      std::lock_guard<std::mutex> lk(g_local_signals_mu);
      auto it = g_local_signals.find((uintptr_t)peer_flag_ptrs[i]);
      if (it != g_local_signals.end()) peer_dev = it->second;
    }
    pt.sys[i] = peer_dev != sig->device;
  }
  return pt;
}

}  // namespace
}  // namespace sg

using namespace sg;

extern "C" {

int32_t sg_signal_create(int32_t device, int32_t nranks, int32_t rank, uint64_t* out_signal) {
  SG_API_BEGIN
  SG_REQUIRE(out_signal, "null out pointer");
  SG_REQUIRE(nranks >= 1 && 0 <= rank && rank < nranks, "rank %d not in [0, %d)", rank, nranks);
  auto s = std::make_unique<Signal>();
  s->device = device;
  s->nranks = nranks;
  s->rank = rank;
  DeviceScope ds(device);
  s->words.alloc(device, s->nwords() * 8);
  SG_CUDA(cudaMemset(s->words.ptr, 0, s->nwords() * 8));
  SG_CUDA(cudaDeviceSynchronize());
  {
    std::lock_guard<std::mutex> lk(g_local_signals_mu);
    g_local_signals[reinterpret_cast<uintptr_t>(s->words.ptr)] = device;
  }
  *out_signal = registry_put(s.release());
  SG_API_END
}

int32_t sg_signal_ptr(uint64_t signal, uint64_t* out_dev_ptr) {
  SG_API_BEGIN
  Signal* s = get<Signal>(signal, ObjKind::Signal);
  SG_REQUIRE(out_dev_ptr, "null out pointer");
  *out_dev_ptr = reinterpret_cast<uint64_t>(s->words.ptr);
  SG_API_END
}

int32_t sg_signal_ipc_handle(uint64_t signal, uint8_t* out_handle, size_t n) {
  SG_API_BEGIN
  Signal* s = get<Signal>(signal, ObjKind::Signal);
  SG_REQUIRE(out_handle && n >= sizeof(cudaIpcMemHandle_t), "buffer must hold %zu bytes", sizeof(cudaIpcMemHandle_t));
  DeviceScope ds(s->device);
  cudaIpcMemHandle_t h;
  SG_CUDA(cudaIpcGetMemHandle(&h, s->words.ptr));
  memcpy(out_handle, &h, sizeof(h));
  SG_API_END
}

int32_t sg_signal_read(uint64_t signal, uint64_t* out_words, int64_t n) {
  SG_API_BEGIN
  Signal* s = get<Signal>(signal, ObjKind::Signal);
  SG_REQUIRE(out_words && n >= (int64_t)s->nwords(), "need %zu words", s->nwords());
  DeviceScope ds(s->device);
  SG_CUDA(cudaMemcpy(out_words, s->words.ptr, s->nwords() * 8, cudaMemcpyDeviceToHost));
  SG_API_END
}

// Overwrite signal words (host -> device, synchronous).  Measurement and tests only: e.g. to
// time one rank's step alone with its owners' ready words already published.
int32_t sg_signal_write(uint64_t signal, const uint64_t* words, int64_t n) {
  SG_API_BEGIN
  Signal* s = get<Signal>(signal, ObjKind::Signal);
  SG_REQUIRE(words && n == (int64_t)s->nwords(), "need exactly %zu words", s->nwords());
  DeviceScope ds(s->device);
  SG_CUDA(cudaMemcpy(s->words.ptr, words, s->nwords() * 8, cudaMemcpyHostToDevice));
  SG_API_END
}

int32_t sg_step_create(uint64_t stencil, uint64_t plan, uint64_t src_field, uint64_t dst_field, uint64_t signal,
                       const uint64_t* peer_ptrs, const int64_t* peer_pitch_elems, const uint64_t* peer_flag_ptrs,
                       uint64_t* out_step) {
  SG_API_BEGIN
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  Plan* p = get<Plan>(plan, ObjKind::Plan);
  Field* src = get<Field>(src_field, ObjKind::Field);
  Field* dst = get<Field>(dst_field, ObjKind::Field);
  Signal* sig = get<Signal>(signal, ObjKind::Signal);
  SG_REQUIRE(out_step, "null out pointer");
  if (src->npts != s->source_nnodes)
    throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: source field has %lld points, weights expect %lld",
                (long long)src->npts, (long long)s->source_nnodes);
  if (dst->npts != s->m)
    throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: target field has %lld points, weights cover %lld",
                (long long)dst->npts, (long long)s->m);
  if (src->levels != dst->levels) throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: level counts differ");
  if (src->npts != p->nnodes)
    throw_error(SG_DOMAIN_ERROR, "PlanMismatch: field has %lld points, plan covers %lld nodes", (long long)src->npts,
                (long long)p->nnodes);
  SG_REQUIRE(src->itemsize == 8 && dst->itemsize == 8, "real64 fields only");
  SG_REQUIRE(src->device == s->device && dst->device == s->device && p->device == s->device &&
                 sig->device == s->device,
             "stencil, plan, fields and signal live on different devices");
  SG_REQUIRE(s->m < INT32_MAX, "too many targets");
  auto st = std::make_unique<Step>();
  st->device = s->device;
  st->signal = signal;
  const PeerTable pt = peer_table(p, sig, peer_ptrs, peer_pitch_elems, peer_flag_ptrs);
  DeviceScope ds(s->device);
  StepArgs& d = st->args;
  d.idx = s->idx.as<int4>();
  d.w = s->w.as<double2>();
  d.m = s->m;
  d.levels = src->levels;
  d.k = s->k;
  d.src = src->buf.as<double>();
  d.src_pitch = src->pitch;
  d.dst = dst->buf.as<double>();
  d.dst_pitch = dst->pitch;
  d.ghost_lo = p->ghost_lo;
  d.ghost_slot = p->ghost_slot.as<int32_t>();
  d.ghost_row = p->ghost_row.as<int32_t>();
  d.flags = sig->words.as<unsigned long long>();
  d.timeout_ns = kTimeoutNs;
  d.nranks = sig->nranks;
  d.rank = sig->rank;
  d.peers = pt;
  // boundary targets (a stencil row >= ghost_lo): the count the last reader checks against
  DevBuf cnt;
  cnt.alloc(s->device, 8);
  SG_CUDA(cudaMemset(cnt.ptr, 0, 8));
  if (s->m) {
    count_boundary<<<(unsigned)((s->m + 255) / 256), 256>>>(d.idx, d.m, d.k, d.ghost_lo,
                                                          cnt.as<unsigned long long>());
    SG_CUDA_LAUNCH();
  }
  unsigned long long nb = 0;
  SG_CUDA(cudaMemcpy(&nb, cnt.ptr, 8, cudaMemcpyDeviceToHost));
  d.n_boundary = (int64_t)nb;
  SG_REQUIRE(nb == 0 || p->recv_off.back() > 0, "stencil reads ghost rows the plan does not receive");
  st->nblocks = std::max<int64_t>(1, (s->m + kWarps - 1) / kWarps);
  *out_step = registry_put(st.release());
  SG_API_END
}

int32_t sg_step_info(uint64_t step, int64_t* out_m, int64_t* out_n_boundary) {
  SG_API_BEGIN
  Step* st = get<Step>(step, ObjKind::Step);
  if (out_m) *out_m = st->args.m;
  if (out_n_boundary) *out_n_boundary = st->args.n_boundary;
  SG_API_END
}

static void step_launch(const uint64_t* steps, int32_t n, int32_t wait_done, uint64_t stream, bool coop) {
  SG_REQUIRE(steps && n >= 1 && n <= kMaxGroup, "1..%d steps per launch", kMaxGroup);
  SG_REQUIRE(coop || !(n > 1 && wait_done),
             "a multi-rank launch on one GPU cannot wait for its own ranks (wait_done=0)");
  Group g{};
  g.n = n;
  g.wait_done = wait_done ? 1 : 0;
  int device = -1, levels = -1;
  g.start[0] = 0;
  for (int i = 0; i < n; ++i) {
    Step* st = get<Step>(steps[i], ObjKind::Step);
    if (i == 0) device = st->device, levels = st->args.levels;
    SG_REQUIRE(st->device == device, "steps of one launch must share a device");
    SG_REQUIRE(st->args.levels == levels, "steps of one launch must share the level count");
    g.d[i] = st->args;
    g.start[i + 1] = g.start[i] + st->nblocks;
  }
  SG_REQUIRE(g.start[n] < INT32_MAX, "too many targets for one launch");
  DeviceScope ds(device);
  cudaStream_t s = as_stream(stream);
  launch_pdl(signal_kernel, 1, kSignalThreads, s, g);
  const unsigned grid = (unsigned)g.start[n];
  switch ((levels + 31) / 32) {
    case 1: launch_pdl(step_kernel<1>, grid, kWarps * 32, s, g, coop); break;
    case 2: launch_pdl(step_kernel<2>, grid, kWarps * 32, s, g, coop); break;
    case 3: launch_pdl(step_kernel<3>, grid, kWarps * 32, s, g, coop); break;
    case 4: launch_pdl(step_kernel<4>, grid, kWarps * 32, s, g, coop); break;
    case 5: launch_pdl(step_kernel<5>, grid, kWarps * 32, s, g, coop); break;
    default: launch_pdl(step_kernel<0>, grid, kWarps * 32, s, g, coop); break;
  }
  SG_CUDA_LAUNCH();
}

int32_t sg_step_launch(const uint64_t* steps, int32_t n, int32_t wait_done, uint64_t stream) {
  SG_API_BEGIN
  step_launch(steps, n, wait_done, stream, false);
  SG_API_END
}

// Every rank of a single-GPU emulation in ONE cooperative launch WITH the tail waits
// (wait_done = 1): all blocks co-resident, so the ranks' last blocks may spin on each other.
// Small problems only (the grid must fit the GPU at once).
int32_t sg_step_launch_cooperative(const uint64_t* steps, int32_t n, uint64_t stream) {
  SG_API_BEGIN
  step_launch(steps, n, 1, stream, true);
  SG_API_END
}

// Bound on every wait of this step (default 10 s); tests shorten it to exercise the timeout.
int32_t sg_step_set_timeout(uint64_t step, uint64_t timeout_ns) {
  SG_API_BEGIN
  Step* st = get<Step>(step, ObjKind::Step);
  SG_REQUIRE(timeout_ns > 0, "timeout must be positive");
  st->args.timeout_ns = timeout_ns;
  SG_API_END
}

// Error word of the step's signal (0 = fine; 1 = an owner never published its rows, 2 = a
// reader never finished) and the last completed epoch.  Synchronous (reads device memory).
int32_t sg_step_check(uint64_t step, uint64_t* out_error, uint64_t* out_epoch) {
  SG_API_BEGIN
  Step* st = get<Step>(step, ObjKind::Step);
  Signal* sig = get<Signal>(st->signal, ObjKind::Signal);
  std::vector<uint64_t> w(sig->nwords());
  DeviceScope ds(sig->device);
  SG_CUDA(cudaMemcpy(w.data(), sig->words.ptr, w.size() * 8, cudaMemcpyDeviceToHost));
  if (out_error) *out_error = w[w_error(sig->nranks)];
  if (out_epoch) *out_epoch = w[w_epoch(sig->nranks)];
  if (w[w_error(sig->nranks)])
    throw_error(SG_DOMAIN_ERROR, "SpheregridError: fused step of rank %d timed out waiting for a peer (%s)", sig->rank,
                w[w_error(sig->nranks)] == 1 ? "owner rows never published" : "reader never finished");
  SG_API_END
}

}  // extern "C"

extern "C" {

int32_t sg_exchange_create(uint64_t plan, uint64_t field, uint64_t signal, const uint64_t* peer_ptrs,
                           const int64_t* peer_pitch_elems, const uint64_t* peer_flag_ptrs, uint64_t* out_exchange) {
  SG_API_BEGIN
  Plan* p = get<Plan>(plan, ObjKind::Plan);
  Field* f = get<Field>(field, ObjKind::Field);
  Signal* sig = get<Signal>(signal, ObjKind::Signal);
  SG_REQUIRE(out_exchange, "null out pointer");
  if (f->npts != p->nnodes)
    throw_error(SG_DOMAIN_ERROR, "PlanMismatch: field has %lld points, plan covers %lld nodes", (long long)f->npts,
                (long long)p->nnodes);
  SG_REQUIRE(f->device == p->device && sig->device == p->device, "plan, field and signal live on different devices");
  SG_REQUIRE(f->itemsize == 4 || f->itemsize == 8, "item size %d", f->itemsize);
  auto x = std::make_unique<Exchange>();
  x->device = p->device;
  x->signal = signal;
  x->itemsize = f->itemsize;
  const PeerTable pt = peer_table(p, sig, peer_ptrs, peer_pitch_elems, peer_flag_ptrs);
  DeviceScope ds(p->device);
  XchgArgs& d = x->args;
  d.base = f->buf.ptr;
  d.pitch = f->pitch;
  d.W = f->levels;
  d.rows = p->recv_rows.as<int32_t>();
  d.remote = p->recv_remote.as<int32_t>();
  d.slot = p->recv_peer.as<int32_t>();
  d.n = p->recv_off.back();
  d.flags = sig->words.as<unsigned long long>();
  d.timeout_ns = kTimeoutNs;
  d.nranks = sig->nranks;
  d.rank = sig->rank;
  d.peers = pt;
  *out_exchange = registry_put(x.release());
  SG_API_END
}

static void exchange_launch(const uint64_t* exchanges, int32_t n, int32_t wait_done, uint64_t stream, bool coop) {
  SG_REQUIRE(exchanges && n >= 1 && n <= kMaxGroup, "1..%d exchanges per launch", kMaxGroup);
  SG_REQUIRE(coop || !(n > 1 && wait_done),
             "a multi-rank launch on one GPU cannot wait for its own ranks (wait_done=0)");
  XGroup g{};
  g.n = n;
  g.wait_done = wait_done ? 1 : 0;

  int device = -1, item = 0, W = 0;
  for (int i = 0; i < n; ++i) {
    Exchange* x = get<Exchange>(exchanges[i], ObjKind::Exchange);
    if (i == 0) device = x->device, item = x->itemsize, W = x->args.W;
    SG_REQUIRE(x->device == device && x->itemsize == item && x->args.W == W,
               "exchanges of one launch must share device, item size and levels");
    g.d[i] = x->args;
  }
  // grid: one block per kXWarps * kXRows ghost rows, at most a resident grid (kXBlocksPerSM
  // blocks per SM) per launch shared among its ranks — each block acquires and counts once;
  // at least one block per rank (it publishes the epoch even without ghosts)
  int nsm = 148;
  SG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  const int64_t cap = std::max<int64_t>(1, (int64_t)nsm * kXBlocksPerSM / n);
  for (int i = 0; i < n; ++i)
    g.start[i + 1] = g.start[i] + std::min<int64_t>(cap, std::max<int64_t>(1, (g.d[i].n + kXWarps * kXRows - 1) /
                                                                                  (kXWarps * kXRows)));
  DeviceScope ds(device);
  cudaStream_t s = as_stream(stream);
  launch_pdl(xsignal_kernel, 1, kSignalThreads, s, g);
  const unsigned grid = (unsigned)g.start[n];
  const int it = (W + 31) / 32;
#define SG_XLAUNCH(Wd)                                                            \
  switch (it) {                                                                   \
    case 1: launch_pdl(xchg_kernel<Wd, 1>, grid, kXWarps * 32, s, g, coop); break;         \
    case 2: launch_pdl(xchg_kernel<Wd, 2>, grid, kXWarps * 32, s, g, coop); break;         \
    case 3: launch_pdl(xchg_kernel<Wd, 3>, grid, kXWarps * 32, s, g, coop); break;         \
    case 4: launch_pdl(xchg_kernel<Wd, 4>, grid, kXWarps * 32, s, g, coop); break;         \
    case 5: launch_pdl(xchg_kernel<Wd, 5>, grid, kXWarps * 32, s, g, coop); break;         \
    default: launch_pdl(xchg_kernel<Wd, 0>, grid, kXWarps * 32, s, g, coop); break;        \
  }
  if (item == 8) {
    SG_XLAUNCH(unsigned long long)
  } else {
    SG_XLAUNCH(unsigned int)
  }
#undef SG_XLAUNCH
  SG_CUDA_LAUNCH();
}

int32_t sg_exchange_launch(const uint64_t* exchanges, int32_t n, int32_t wait_done, uint64_t stream) {
  SG_API_BEGIN
  exchange_launch(exchanges, n, wait_done, stream, false);
  SG_API_END
}

int32_t sg_exchange_launch_cooperative(const uint64_t* exchanges, int32_t n, uint64_t stream) {
  SG_API_BEGIN
  exchange_launch(exchanges, n, 1, stream, true);
  SG_API_END
}

int32_t sg_exchange_set_timeout(uint64_t exchange, uint64_t timeout_ns) {
  SG_API_BEGIN
  Exchange* x = get<Exchange>(exchange, ObjKind::Exchange);
  SG_REQUIRE(timeout_ns > 0, "timeout must be positive");
  x->args.timeout_ns = timeout_ns;
  SG_API_END
}

int32_t sg_exchange_signal(uint64_t exchange, uint64_t* out_signal) {
  SG_API_BEGIN
  Exchange* x = get<Exchange>(exchange, ObjKind::Exchange);
  SG_REQUIRE(out_signal, "null out pointer");
  *out_signal = x->signal;
  SG_API_END
}

}  // extern "C"
