// The host-buffer execute (sg_remap_execute_host): apply_remap with HOST source and target
// arrays (interp.py:206-228), pipelined over source-row chunks on three streams — h2d of a
// chunk, apply of the targets whose stencils are complete, d2h of their rows — in four modes:
// dma (copy the referenced row runs), compact (pack only referenced rows on the host with
// non-temporal stores into a pinned ring; apply from a compact device copy with a renumbered
// stencil), gather (the same compact device copy, filled by a GPU kernel that reads only the
// referenced rows straight out of the pinned, mapped user array: no host CPU work, no DMA of
// unreferenced rows) and zero-copy (the apply kernel reads/writes pinned host memory directly).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <emmintrin.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "apply_internal.cuh"
#include "host_pool.h"
#include "tma.cuh"

namespace sg {
namespace {
using namespace detail;

struct CompactRun {
  int64_t src, len, dst;  // source row, rows, compact row
};

struct HostPlan {
  int nchunks = 0;
  bool host_tables = false;  // idx_host / mark_host / runs / t_end built on the host
  bool device_gather = false;  // gather-mode tables (t_end, cb, cidx, pieces) built on the device
  std::vector<int64_t> t_end;                                  // chunk c: targets [t_end[c-1], t_end[c])
  std::vector<std::vector<std::pair<int64_t, int64_t>>> runs;  // chunk c: referenced source rows
  int64_t rows_copied = 0;
  cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
  cudaStream_t s_in2 = nullptr;  // gather mode: odd chunks' gathers (overlaps consecutive gathers' tails)
  std::vector<cudaEvent_t> ev_in, ev_cmp;
  std::vector<int4> idx_host;           // stencil copy (compact rebuilds)
  std::vector<unsigned char> mark_host; // referenced source rows
  // compact mode: only referenced rows cross PCIe, packed on the host into pinned staging
  bool compact_ready = false;
  int period = -1;                                // every period-th chunk is copied directly
  int64_t ncompact = 0;                           // device rows of the compact source
  std::vector<std::vector<CompactRun>> cruns;     // chunk c: exact referenced runs (packed chunks)
  std::vector<int64_t> cb;                        // chunk c: device rows [cb[c], cb[c+1])
  std::vector<char> direct;                       // chunk c copied straight from the user array
  std::vector<int64_t> rlo;                       // chunk c: first source row
  DevBuf cidx;                                    // int4[m]: stencil in compact row numbering
  DevBuf gsrc;                                    // int32[ncompact]: source row of each compact row
  // gather mode, TMA path: referenced runs cut into pieces of <= piece_rows rows
  int piece_levels = -1, piece_rows = 0;
  std::vector<int64_t> pb;                        // chunk c: pieces [pb[c], pb[c+1])
  DevBuf pieces;                                  // int2 (first source row, rows) per piece
  DevBuf pdst;                                    // int64 first compact row per piece
  std::vector<std::unique_ptr<DevBuf>> csrc;      // per field: U compact rows on the device
  static constexpr int kRing = 3;
  std::vector<void*> ring;                        // per (field, slot): pinned staging
  size_t ring_bytes = 0;
  int ring_fields = 0;
  ~HostPlan() {
    for (void* p : ring)
      if (p) cudaFreeHost(p);
  }
};

// Row copy into the pinned staging ring with non-temporal 8-B stores (movnti): the staging
// lines are not read for ownership, cutting host memory traffic of the packing by a third.
inline void copy_rows_nt(char* dst, const char* src, size_t bytes) {
  // 8-B aligned rows: one movnti to reach 16-B destination alignment, then 16-B streams
  size_t off = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) && bytes >= 8) {
    _mm_stream_si64(reinterpret_cast<long long*>(dst), *reinterpret_cast<const long long*>(src));
    off = 8;
  }
  for (; off + 16 <= bytes; off += 16)
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + off), _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + off)));
  for (; off + 8 <= bytes; off += 8)
    _mm_stream_si64(reinterpret_cast<long long*>(dst + off), *reinterpret_cast<const long long*>(src + off));
}

// gather mode, TMA path (the default): one producer thread per CTA bulk-copies the 16-B
// aligned superset of a piece (a run of consecutive referenced source rows, <= piece_rows
// rows) out of the mapped host array into a shared-memory ring stage; 4 consumer warps copy
// the stage into the piece's compact rows.  The copy engine of the TMA unit issues larger PCIe
// reads than warp loads: tools/probes/pcie_gather_probe.cu measured 50.5 GB/s vs 48.6 for the
// warp-per-row gather below (DMA of every row: 55.6 GB/s, but on 1/0.77 more bytes).
constexpr int kGatherStages = 4;
constexpr int kGatherStreams = 1;
constexpr int kGatherCtasPerSM = 4;  // 113.8-114.6 ms vs 115.3-115.6 at 2 (profiles/r02_e2e_gather_knobs.jsonl)

int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  const int x = atoi(v);
  return x < lo ? lo : (x > hi ? hi : x);
}
constexpr int kGatherPieceDoubles = 12 * 137;  // ~13 KB per stage

__global__ void __launch_bounds__(160) gather_tma(const double* __restrict__ host, int64_t host_rows,
                                                  const int2* __restrict__ pieces, const int64_t* __restrict__ pdst,
                                                  double* __restrict__ out, int64_t p0, int64_t p1, int levels,
                                                  int slot) {
  using namespace tma;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + kGatherStages;
  double* ring = reinterpret_cast<double*>(smem_raw + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uintptr_t lo = reinterpret_cast<uintptr_t>(host);
  const uintptr_t hi = reinterpret_cast<uintptr_t>(host + host_rows * levels);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGatherStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 4) {  // producer
    if (lane != 0) return;
    int it = 0;
    for (int64_t p = p0 + blockIdx.x; p < p1; p += gridDim.x, ++it) {
      const int st = it % kGatherStages;
      if (it >= kGatherStages) mbar_wait(&empty[st], ((it / kGatherStages) - 1) & 1);
      const int2 pc = __ldg(pieces + p);
      const uintptr_t a = reinterpret_cast<uintptr_t>(host + (int64_t)pc.x * levels);
      const uintptr_t s0 = a & ~uintptr_t(15), s1 = (a + (uintptr_t)pc.y * levels * 8 + 15) & ~uintptr_t(15);
      if (s0 < lo || s1 > hi) {  // superset leaves the array: consumers load this piece directly
        mbar_arrive(&full[st]);
      } else {
        mbar_expect_tx(&full[st], (uint32_t)(s1 - s0));
        bulk_g2s(ring + (size_t)st * slot, reinterpret_cast<const void*>(s0), (uint32_t)(s1 - s0), &full[st]);
      }
    }
    return;
  }
  int it = 0;
  for (int64_t p = p0 + blockIdx.x; p < p1; p += gridDim.x, ++it) {
    const int st = it % kGatherStages;
    const int2 pc = __ldg(pieces + p);
    double* d = out + __ldg(pdst + p) * levels;
    const double* src = host + (int64_t)pc.x * levels;
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uintptr_t s0 = a & ~uintptr_t(15), s1 = (a + (uintptr_t)pc.y * levels * 8 + 15) & ~uintptr_t(15);
    const bool direct = s0 < lo || s1 > hi;
    const double* b = direct ? src : ring + (size_t)st * slot + ((a - s0) >> 3);
    const int n = pc.y * levels;
    mbar_wait(&full[st], (it / kGatherStages) & 1);
    for (int i = threadIdx.x; i < n; i += 128) d[i] = b[i];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

// warp-per-row gather (levels too large for a ring stage): compact rows [u0, u1) <- host
// rows gsrc[u], every load of the row in flight before the stores (PCIe read latency)
template <int IT>
__global__ void __launch_bounds__(256) gather_rows(const double* __restrict__ host, const int32_t* __restrict__ gsrc,
                                                   double* __restrict__ out, int64_t u0, int64_t u1, int levels) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = u0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); u < u1; u += stride) {
    const double* src = host + (int64_t)__ldg(gsrc + u) * levels;
    double* dst = out + u * levels;
    if constexpr (IT == 0) {
      for (int l = lane; l < levels; l += 32) dst[l] = src[l];
    } else {
      double v[IT];
#pragma unroll
      for (int i = 0; i < IT; ++i)
        if (lane + 32 * i < levels) v[i] = src[lane + 32 * i];
#pragma unroll
      for (int i = 0; i < IT; ++i)
        if (lane + 32 * i < levels) dst[lane + 32 * i] = v[i];
    }
  }
}

// 4 of the 8 resident 256-thread blocks per SM: leaves room for the apply of the previous
// chunk, which runs concurrently on its own stream
void launch_gather_rows(const double* host, const int32_t* gsrc, double* out, int64_t u0, int64_t u1, int levels,
                        cudaStream_t st) {
  if (u1 <= u0) return;
  const unsigned grid = (unsigned)std::min<int64_t>((u1 - u0 + 7) / 8, 148 * 4);
  switch ((levels + 31) / 32) {
    case 1: gather_rows<1><<<grid, 256, 0, st>>>(host, gsrc, out, u0, u1, levels); break;
    case 2: gather_rows<2><<<grid, 256, 0, st>>>(host, gsrc, out, u0, u1, levels); break;
    case 3: gather_rows<3><<<grid, 256, 0, st>>>(host, gsrc, out, u0, u1, levels); break;
    case 4: gather_rows<4><<<grid, 256, 0, st>>>(host, gsrc, out, u0, u1, levels); break;
    case 5: gather_rows<5><<<grid, 256, 0, st>>>(host, gsrc, out, u0, u1, levels); break;
    default: gather_rows<0><<<grid, 256, 0, st>>>(host, gsrc, out, u0, u1, levels); break;
  }
  SG_CUDA_LAUNCH();
}

int gather_slot(int levels, int piece_rows) { return (piece_rows * levels + 2 + 1) & ~1; }  // doubles, 16-B multiple

}  // namespace

namespace detail {
int gather_piece_rows(int levels) { return std::max(1, kGatherPieceDoubles / levels); }
bool gather_fits(int levels) { return (size_t)levels * 8 + 16 <= (size_t)kGatherPieceDoubles * 8; }

void launch_gather_tma(const double* host, int64_t host_rows, const int2* pieces, const int64_t* pdst, double* out,
                       int64_t p0, int64_t p1, int levels, int piece_rows, cudaStream_t st, int ctas_per_sm) {
  if (p1 <= p0) return;
  const int slot = gather_slot(levels, piece_rows);
  const size_t smem = 128 + (size_t)kGatherStages * slot * 8;
  SG_CUDA(cudaFuncSetAttribute(gather_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // ctas_per_sm CTAs per SM (4 stages x ~13 KB each; 4 x 53 KB fit): the apply of the
  // previous chunk (no shared memory) co-resides
  const unsigned grid = (unsigned)std::min<int64_t>(p1 - p0, 148 * ctas_per_sm);
  gather_tma<<<grid, 160, smem, st>>>(host, host_rows, pieces, pdst, out, p0, p1, levels, slot);
  SG_CUDA_LAUNCH();
}
}  // namespace detail

namespace {

HostPool& host_pool() {
  static HostPool pool(std::max(1u, std::min(32u, std::thread::hardware_concurrency())) - 1);
  return pool;
}

// Device layout of the compact source: chunk by chunk, a packed chunk contributes its
// referenced rows, a direct chunk (every `period`-th, period > 0) its whole row range, which
// one DMA copies straight from the user's array — the split balances host packing bandwidth
// against PCIe bytes.  The stencil is renumbered into that layout.
void build_compact(Stencil* s, HostPlan* hp, const std::vector<int4>& idx, const std::vector<unsigned char>& mark,
                   int period) {
  const int64_t n = s->source_nnodes, m = s->m;
  std::vector<int32_t> cpos((size_t)n, -1);
  hp->cruns.assign(hp->nchunks, {});
  hp->cb.assign(hp->nchunks + 1, 0);
  hp->direct.assign(hp->nchunks, 0);
  hp->rlo.assign(hp->nchunks + 1, 0);
  int64_t rprev = 0, u = 0;
  for (int c = 0; c < hp->nchunks; ++c) {
    const int64_t rb = (c + 1 == hp->nchunks) ? n : n * (c + 1) / hp->nchunks;
    hp->rlo[c] = rprev;
    hp->cb[c] = u;
    if (period > 0 && c % period == period - 1) {
      hp->direct[c] = 1;
      for (int64_t i = rprev; i < rb; ++i) cpos[i] = (int32_t)(u + (i - rprev));
      u += rb - rprev;
    } else {
      int64_t i = rprev;
      while (i < rb) {
        while (i < rb && !mark[i]) ++i;
        if (i >= rb) break;
        int64_t j = i;
        while (j < rb && mark[j]) ++j;
        hp->cruns[c].push_back(CompactRun{i, j - i, u});
        for (int64_t q = i; q < j; ++q) cpos[q] = (int32_t)u++;
        i = j;
      }
    }
    rprev = rb;
  }
  hp->rlo[hp->nchunks] = n;
  hp->cb[hp->nchunks] = u;
  hp->ncompact = u;
  std::vector<int4> ci((size_t)m);
  for (int64_t t = 0; t < m; ++t) {
    const int4 id = idx[t];
    ci[t] = make_int4(cpos[id.x], cpos[id.y], cpos[id.z], s->k == 4 ? cpos[id.w] : 0);
  }
  hp->cidx.alloc(s->device, std::max<size_t>(ci.size(), 1) * sizeof(int4));
  if (m) SG_CUDA(cudaMemcpy(hp->cidx.ptr, ci.data(), ci.size() * sizeof(int4), cudaMemcpyHostToDevice));
  std::vector<int32_t> gs((size_t)u);
  for (int c = 0; c < hp->nchunks; ++c) {
    if (hp->direct[c])
      for (int64_t i = hp->rlo[c]; i < hp->rlo[c + 1]; ++i) gs[(size_t)(hp->cb[c] + i - hp->rlo[c])] = (int32_t)i;
    for (const auto& r : hp->cruns[c])
      for (int64_t q = 0; q < r.len; ++q) gs[(size_t)(r.dst + q)] = (int32_t)(r.src + q);
  }
  hp->gsrc.alloc(s->device, std::max<size_t>(gs.size(), 1) * sizeof(int32_t));
  if (u) SG_CUDA(cudaMemcpy(hp->gsrc.ptr, gs.data(), gs.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  hp->period = period;
  hp->compact_ready = true;
}

std::mutex g_plan_mu;

HostPlan* host_plan(Stencil* s, int nchunks) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto* hp = static_cast<HostPlan*>(s->host_plan);
  if (hp && hp->nchunks == nchunks) return hp;
  s->destroy_host_plan();
  auto owned = std::make_unique<HostPlan>();
  hp = owned.get();
  hp->nchunks = nchunks;
  SG_CUDA(cudaStreamCreateWithFlags(&hp->s_in, cudaStreamNonBlocking));
  SG_CUDA(cudaStreamCreateWithFlags(&hp->s_cmp, cudaStreamNonBlocking));
  SG_CUDA(cudaStreamCreateWithFlags(&hp->s_out, cudaStreamNonBlocking));
  SG_CUDA(cudaStreamCreateWithFlags(&hp->s_in2, cudaStreamNonBlocking));
  hp->ev_in.resize(nchunks);
  hp->ev_cmp.resize(nchunks);
  for (int c = 0; c < nchunks; ++c) {
    SG_CUDA(cudaEventCreateWithFlags(&hp->ev_in[c], cudaEventDisableTiming));
    SG_CUDA(cudaEventCreateWithFlags(&hp->ev_cmp[c], cudaEventDisableTiming));
  }
  s->host_plan = owned.release();
  return hp;
}

// Host-side tables of the dma / compact modes: the stencil copied down, referenced rows,
// the target ranges each chunk of source rows completes, referenced runs per chunk.
void host_tables(Stencil* s, HostPlan* hp) {
  if (hp->host_tables) return;
  const int nchunks = hp->nchunks;
  const int64_t m = s->m, n = s->source_nnodes;
  std::vector<int4> idx((size_t)m);
  if (m) SG_CUDA(cudaMemcpy(idx.data(), s->idx.ptr, (size_t)m * sizeof(int4), cudaMemcpyDeviceToHost));
  std::vector<unsigned char> mark((size_t)n, 0);
  std::vector<int64_t> pmax((size_t)m);
  int64_t run_max = -1;
  for (int64_t t = 0; t < m; ++t) {
    const int4 id = idx[t];
    mark[id.x] = mark[id.y] = mark[id.z] = 1;
    run_max = std::max<int64_t>(run_max, std::max(id.x, std::max(id.y, id.z)));
    if (s->k == 4) {
      mark[id.w] = 1;
      run_max = std::max<int64_t>(run_max, id.w);
    }
    pmax[t] = run_max;  // monotone: targets [0, t] need source rows <= pmax[t]
  }
  int64_t tprev = 0, rprev = 0;
  hp->t_end.assign(nchunks, 0);
  hp->runs.assign(nchunks, {});
  hp->rows_copied = 0;
  for (int c = 0; c < nchunks; ++c) {
    const int64_t rb = (c + 1 == nchunks) ? n : n * (c + 1) / nchunks;  // source rows [rprev, rb)
    int64_t te = (c + 1 == nchunks) ? m : (int64_t)(std::lower_bound(pmax.begin(), pmax.end(), rb) - pmax.begin());
    te = std::max(te, tprev);
    hp->t_end[c] = te;
    // referenced runs of [rprev, rb); unreferenced gaps shorter than 64 rows are copied through
    int64_t i = rprev;
    while (i < rb) {
      while (i < rb && !mark[i]) ++i;
      if (i >= rb) break;
      int64_t j = i;
      for (;;) {
        while (j < rb && mark[j]) ++j;
        int64_t g = j;
        while (g < rb && !mark[g] && g - j < 64) ++g;
        if (g < rb && mark[g]) j = g;  // short gap: merge
        else break;
      }
      hp->runs[c].emplace_back(i, j);
      hp->rows_copied += j - i;
      i = j;
    }
    tprev = te;
    rprev = rb;
  }
  hp->idx_host = std::move(idx);
  hp->mark_host = std::move(mark);
  hp->host_tables = true;
}

// ---- gather-mode tables built on the device (the default host-field path) ---------------------
// Same layout as host_tables + build_compact(period 0) on the host: compact row of a
// referenced source row = exclusive scan of the referenced flags; pieces = maximal runs of
// referenced rows inside a chunk of source rows, cut every piece_rows rows; t_end[c] = first
// target whose prefix-max stencil row reaches the next chunk.  ~10 ms instead of ~180 ms of
// host loops and pageable uploads at cfg3 (first call of apply_remap on host fields).
__global__ void plan_mark(const int4* idx, int64_t m, int k, int32_t* mark, int32_t* tmax) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int4 id = idx[t];
  mark[id.x] = 1;
  mark[id.y] = 1;
  mark[id.z] = 1;
  int hi = max(id.x, max(id.y, id.z));
  if (k == 4) {
    mark[id.w] = 1;
    hi = max(hi, id.w);
  }
  tmax[t] = hi;
}

struct MaxOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

__device__ __forceinline__ int64_t chunk_lo(int64_t n, int nchunks, int c) { return n * c / nchunks; }

// candidate segment start of row i (a referenced row that starts a run or a chunk), else -1
__global__ void plan_starts(const int32_t* mark, int64_t n, int nchunks, int32_t* cand) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool start = false;
  if (mark[i]) {
    // chunk c holds rows [n*c/nchunks, n*(c+1)/nchunks); i starts a chunk iff i == chunk_lo(c(i))
    int c = (int)((i * nchunks) / n);
    while (c + 1 < nchunks && chunk_lo(n, nchunks, c + 1) <= i) ++c;
    while (c > 0 && chunk_lo(n, nchunks, c) > i) --c;
    start = i == 0 || !mark[i - 1] || i == chunk_lo(n, nchunks, c);
  }
  cand[i] = start ? (int32_t)i : -1;
}

__global__ void plan_piece_flags(const int32_t* mark, const int32_t* seg, int64_t n, int prows,
                                 unsigned char* flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = mark[i] && ((i - seg[i]) % prows == 0);
}

__global__ void plan_pieces(const int32_t* starts, int64_t np, const int32_t* seg, const int32_t* cpos,
                            const int32_t* mark, int64_t n, int nchunks, int prows, int2* pieces,
                            int64_t* pdst) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int32_t st = starts[k];
  int len = 1;
  while (len < prows && st + len < n && mark[st + len] && seg[st + len] == seg[st]) ++len;
  pieces[k] = make_int2(st, len);
  pdst[k] = cpos[st];
}

__global__ void plan_cidx(const int4* idx, int64_t m, int k, const int32_t* cpos, int4* cidx) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int4 id = idx[t];
  cidx[t] = make_int4(cpos[id.x], cpos[id.y], cpos[id.z], k == 4 ? cpos[id.w] : 0);
}

// per chunk c: t_end (first target t with pmax[t] >= rb_c), cb = cpos[rlo_c], pb = first piece
// starting at or after rlo_c
__global__ void plan_chunks(const int32_t* pmax, int64_t m, const int32_t* cpos, const int32_t* starts, int64_t np,
                            int64_t n, int nchunks, int64_t* t_end, int64_t* cb, int64_t* pb) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nchunks) return;
  const int64_t lo = c == nchunks ? n : chunk_lo(n, nchunks, c);
  cb[c] = cpos[lo];
  int64_t a = 0, b = np;  // first piece with start >= lo
  while (a < b) {
    const int64_t mid = (a + b) / 2;
    if (starts[mid] < lo) a = mid + 1; else b = mid;
  }
  pb[c] = a;
  if (c < nchunks) {
    const int64_t rb = c + 1 == nchunks ? n : chunk_lo(n, nchunks, c + 1);
    int64_t x = 0, y = m;  // lower_bound(pmax, rb)
    while (x < y) {
      const int64_t mid = (x + y) / 2;
      if (pmax[mid] < rb) x = mid + 1; else y = mid;
    }
    t_end[c] = c + 1 == nchunks ? m : x;
  }
}

struct PlanBuf {  // a slice of the plan's temporary arena
  void* ptr;
  size_t bytes;
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

void device_gather_tables(Stencil* s, HostPlan* hp, int levels, cudaStream_t st) {
  const int prows = gather_piece_rows(levels);
  if (hp->device_gather && hp->piece_rows == prows) return;
  const int nchunks = hp->nchunks;
  const int64_t m = s->m, n = s->source_nnodes;
  SG_REQUIRE(n < INT32_MAX && m < INT32_MAX, "too large for the device plan");
  const int dev = s->device;
  // one arena for every temporary (a cudaMalloc per buffer cost ~10 ms each here)
  struct Part {
    size_t off, bytes;
  };
  size_t arena_bytes = 0;
  auto part = [&](size_t bytes) {
    Part p{arena_bytes, bytes};
    arena_bytes += (bytes + 255) / 256 * 256;
    return p;
  };
  const size_t nn = (size_t)std::max<int64_t>(n, 1), mm = (size_t)std::max<int64_t>(m, 1);
  const Part p_mark = part((nn + 1) * 4), p_tmax = part(mm * 4), p_pmax = part(mm * 4), p_cpos = part((nn + 1) * 4),
             p_cand = part(nn * 4), p_seg = part(nn * 4), p_flag = part(nn), p_starts = part(nn * 4), p_nsel = part(8),
             p_tend = part((size_t)nchunks * 8), p_cb = part((size_t)(nchunks + 1) * 8),
             p_pb = part((size_t)(nchunks + 1) * 8);
  // CUB temp storage: sized with null pointers first
  size_t b1 = 0, b2 = 0, b3 = 0, b4 = 0;
  SG_CUDA(cub::DeviceScan::InclusiveScan(nullptr, b1, (int32_t*)nullptr, (int32_t*)nullptr, MaxOp(), (int)mm, st));
  SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b2, (int32_t*)nullptr, (int32_t*)nullptr, (int)(nn + 1), st));
  SG_CUDA(cub::DeviceScan::InclusiveScan(nullptr, b3, (int32_t*)nullptr, (int32_t*)nullptr, MaxOp(), (int)nn, st));
  SG_CUDA(cub::DeviceSelect::Flagged(nullptr, b4, thrust::counting_iterator<int32_t>(0), (unsigned char*)nullptr,
                                     (int32_t*)nullptr, (int64_t*)nullptr, (int)nn, st));
  const Part p_tmp = part(std::max(std::max(b1, b2), std::max(b3, b4)) + 16);
  DevBuf arena;
  arena.alloc(dev, arena_bytes);
  auto buf = [&](Part p) { return PlanBuf{arena.as<char>() + p.off, p.bytes}; };
  const PlanBuf mark = buf(p_mark), tmax = buf(p_tmax), pmax = buf(p_pmax), cpos = buf(p_cpos), cand = buf(p_cand),
            seg = buf(p_seg), flag = buf(p_flag), starts = buf(p_starts), nsel = buf(p_nsel), t_end = buf(p_tend),
            cb = buf(p_cb), pb = buf(p_pb), tmp = buf(p_tmp);
  SG_CUDA(cudaMemsetAsync(mark.ptr, 0, mark.bytes, st));
  const unsigned gm = (unsigned)((m + 255) / 256), gn = (unsigned)((n + 255) / 256);
  if (m) plan_mark<<<gm, 256, 0, st>>>(s->idx.as<int4>(), m, s->k, mark.as<int32_t>(), tmax.as<int32_t>());
  SG_CUDA_LAUNCH();
  size_t tb = tmp.bytes;
  if (m) SG_CUDA(cub::DeviceScan::InclusiveScan(tmp.ptr, tb, tmax.as<int32_t>(), pmax.as<int32_t>(), MaxOp(), (int)m, st));
  tb = tmp.bytes;  // mark[n] is the zero pad: cpos[n] = U
  SG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tb, mark.as<int32_t>(), cpos.as<int32_t>(), (int)(n + 1), st));
  if (n) {
    plan_starts<<<gn, 256, 0, st>>>(mark.as<int32_t>(), n, nchunks, cand.as<int32_t>());
    SG_CUDA_LAUNCH();
    tb = tmp.bytes;
    SG_CUDA(cub::DeviceScan::InclusiveScan(tmp.ptr, tb, cand.as<int32_t>(), seg.as<int32_t>(), MaxOp(), (int)n, st));
    plan_piece_flags<<<gn, 256, 0, st>>>(mark.as<int32_t>(), seg.as<int32_t>(), n, prows, flag.as<unsigned char>());
    SG_CUDA_LAUNCH();
    tb = tmp.bytes;
    SG_CUDA(cub::DeviceSelect::Flagged(tmp.ptr, tb, thrust::counting_iterator<int32_t>(0), flag.as<unsigned char>(),
                                       starts.as<int32_t>(), nsel.as<int64_t>(), (int)n, st));
  } else {
    SG_CUDA(cudaMemsetAsync(nsel.ptr, 0, 8, st));
  }
  int64_t np = 0;
  int32_t U = 0;
  SG_CUDA(cudaMemcpyAsync(&np, nsel.ptr, 8, cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaMemcpyAsync(&U, cpos.as<int32_t>() + n, 4, cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  hp->pieces.alloc(dev, (size_t)std::max<int64_t>(np, 1) * sizeof(int2));
  hp->pdst.alloc(dev, (size_t)std::max<int64_t>(np, 1) * sizeof(int64_t));
  hp->cidx.alloc(dev, (size_t)std::max<int64_t>(m, 1) * sizeof(int4));
  if (np) {
    plan_pieces<<<(unsigned)((np + 255) / 256), 256, 0, st>>>(starts.as<int32_t>(), np, seg.as<int32_t>(),
                                                             cpos.as<int32_t>(), mark.as<int32_t>(), n, nchunks,
                                                             prows, hp->pieces.as<int2>(), hp->pdst.as<int64_t>());
    SG_CUDA_LAUNCH();
  }
  if (m) {
    plan_cidx<<<gm, 256, 0, st>>>(s->idx.as<int4>(), m, s->k, cpos.as<int32_t>(), hp->cidx.as<int4>());
    SG_CUDA_LAUNCH();
  }
  plan_chunks<<<(nchunks + 1 + 127) / 128, 128, 0, st>>>(pmax.as<int32_t>(), m, cpos.as<int32_t>(),
                                                        starts.as<int32_t>(), np, n, nchunks, t_end.as<int64_t>(),
                                                        cb.as<int64_t>(), pb.as<int64_t>());
  SG_CUDA_LAUNCH();
  std::vector<int64_t> te(nchunks);
  hp->cb.assign(nchunks + 1, 0);
  hp->pb.assign(nchunks + 1, 0);
  SG_CUDA(cudaMemcpyAsync(te.data(), t_end.ptr, (size_t)nchunks * 8, cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaMemcpyAsync(hp->cb.data(), cb.ptr, (size_t)(nchunks + 1) * 8, cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaMemcpyAsync(hp->pb.data(), pb.ptr, (size_t)(nchunks + 1) * 8, cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  int64_t tprev = 0;
  hp->t_end.assign(nchunks, 0);
  for (int c = 0; c < nchunks; ++c) hp->t_end[c] = tprev = std::max(te[c], tprev);
  hp->ncompact = U;
  hp->direct.assign(nchunks, 0);
  hp->piece_levels = levels;
  hp->piece_rows = prows;
  hp->period = 0;
  hp->compact_ready = false;  // the host compact tables (cruns, gsrc) are not built
  hp->device_gather = true;
}

}  // namespace

void Stencil::destroy_host_plan() {
  auto* hp = static_cast<HostPlan*>(host_plan);
  if (!hp) return;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != device) cudaSetDevice(device);
  for (auto e : hp->ev_in) cudaEventDestroy(e);
  for (auto e : hp->ev_cmp) cudaEventDestroy(e);
  if (hp->s_in) cudaStreamDestroy(hp->s_in);
  if (hp->s_cmp) cudaStreamDestroy(hp->s_cmp);
  if (hp->s_out) cudaStreamDestroy(hp->s_out);
  if (hp->s_in2) cudaStreamDestroy(hp->s_in2);
  if (cur != device && cur >= 0) cudaSetDevice(cur);
  delete hp;
  host_plan = nullptr;
}

}  // namespace sg

using namespace sg;
using namespace sg::detail;

extern "C" {

int32_t sg_remap_execute_host(uint64_t stencil, const uint64_t* src_fields, const uint64_t* dst_fields,
                              int32_t nfields, const uint64_t* host_src, const uint64_t* host_dst, int32_t nchunks,
                              int32_t variant, int32_t flags, int64_t* out_rows_copied) {
  SG_API_BEGIN
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  FieldPairs p = check_pairs(s, src_fields, dst_fields, nfields);
  SG_REQUIRE(host_src && host_dst, "null host arrays");
  for (int f = 0; f < nfields; ++f) {
    SG_REQUIRE(host_src[f] && host_dst[f], "null host array for field %d", f);
    SG_REQUIRE(p.src[f]->pitch == p.levels && p.dst[f]->pitch == p.levels, "execute_host needs dense fields");
  }
  SG_REQUIRE(nchunks >= 1 && nchunks <= 1024, "nchunks must be in [1, 1024]");
  DeviceScope ds(s->device);
  const size_t row = (size_t)p.levels * 8;
  // device addresses of pinned, mapped host arrays (zero-copy and gather modes)
  auto mapped = [](uint64_t host, const char* mode) -> void* {
    cudaPointerAttributes at{};
    SG_CUDA(cudaPointerGetAttributes(&at, reinterpret_cast<const void*>(host)));
    SG_REQUIRE(at.type == cudaMemoryTypeHost && at.devicePointer,
               "%s execute needs pinned, mapped host arrays (sg_host_alloc / sg_host_register)", mode);
    return at.devicePointer;
  };
  if (flags & 2) {
    // zero-copy: the apply kernel reads the referenced source rows straight out of pinned
    // host memory over PCIe and streams the target rows back into pinned host memory — no
    // staging, no DMA engine, only referenced rows cross the link (U/n = 77 % at cfg3)
    std::vector<const double*> hs(nfields);
    std::vector<double*> hd(nfields);
    for (int f = 0; f < nfields; ++f) {
      hs[f] = static_cast<const double*>(mapped(host_src[f], "zero-copy"));
      hd[f] = static_cast<double*>(mapped(host_dst[f], "zero-copy"));
    }
    cudaStream_t st = 0;
    for (int f0 = 0; f0 < nfields; f0 += kMaxFields) {
      ApplyArgs a = make_args(s, p, f0, 0, s->m);
      for (int f = 0; f < a.nfields; ++f) {
        a.src[f] = hs[f0 + f];
        a.dst[f] = hd[f0 + f];
        a.src_pitch[f] = a.dst_pitch[f] = p.levels;
      }
      launch_apply(a, variant == 2 ? 0 : variant, st);
    }
    SG_CUDA(cudaStreamSynchronize(st));
    if (out_rows_copied) *out_rows_copied = s->distinct_sources;
    return SG_OK;
  }
  HostPlan* hp = host_plan(s, nchunks);
  const bool gather = (flags & 4) != 0;
  const bool compact = (flags & 1) != 0 || gather;
  // TMA ring stage must hold at least one 16-B aligned row superset; flags bit 3 forces the
  // warp-per-row gather (kept for comparison)
  const bool tma_gather = gather && !(flags & 8) && gather_fits(p.levels);
  // measurement knobs of the gather pipeline (tools/e2e_sweep.py): gather streams, CTAs per SM
  const int gather_streams = env_int("SG_GATHER_STREAMS", kGatherStreams, 1, 2);
  const int gather_ctas = env_int("SG_GATHER_CTAS", kGatherCtasPerSM, 1, 8);
  std::vector<const double*> gsrc_host(gather ? nfields : 0);
  for (int f = 0; f < (int)gsrc_host.size(); ++f)
    gsrc_host[f] = static_cast<const double*>(mapped(host_src[f], "gather"));
  if (tma_gather) {
    device_gather_tables(s, hp, p.levels, hp->s_in);  // the default path: tables built on the GPU
  } else {
    host_tables(s, hp);
    if (compact) {
      const int period = gather ? 0 : (flags >> 8) & 0xff;
      if (!hp->compact_ready || hp->period != period) {
        build_compact(s, hp, hp->idx_host, hp->mark_host, period);
        hp->device_gather = false;
      }
      // the pinned staging ring (sized for the largest chunk)
      size_t maxc = 0;
      for (int c = 0; c < nchunks; ++c)
        if (!hp->direct[c]) maxc = std::max<size_t>(maxc, (size_t)(hp->cb[c + 1] - hp->cb[c]));
      const size_t need = std::max<size_t>(maxc * row, 16);
      if (!gather && (hp->ring_bytes < need || hp->ring_fields < nfields)) {
        for (void* q : hp->ring)
          if (q) cudaFreeHost(q);
        hp->ring.assign((size_t)nfields * HostPlan::kRing, nullptr);
        for (auto& q : hp->ring) SG_CUDA(cudaHostAlloc(&q, need, cudaHostAllocPortable));
        hp->ring_bytes = need;
        hp->ring_fields = nfields;
      }
    }
  }
  if (compact) {  // device compact sources
    while ((int)hp->csrc.size() < nfields) hp->csrc.emplace_back(new DevBuf());
    for (int f = 0; f < nfields; ++f)
      if (hp->csrc[f]->bytes < std::max<size_t>(hp->ncompact * row, 16))
        hp->csrc[f]->alloc(s->device, std::max<size_t>(hp->ncompact * row, 16));
  }
  int64_t tprev = 0, copied = 0;
  for (int c = 0; c < nchunks; ++c) {
    if (compact) {
      if (hp->direct[c]) {  // whole row range straight from the user's array
        const int64_t nrows = hp->rlo[c + 1] - hp->rlo[c];
        for (int f = 0; f < nfields; ++f)
          if (nrows)
            SG_CUDA(cudaMemcpyAsync(hp->csrc[f]->as<char>() + hp->cb[c] * row,
                                    reinterpret_cast<const char*>(host_src[f]) + hp->rlo[c] * row, (size_t)nrows * row,
                                    cudaMemcpyHostToDevice, hp->s_in));
        copied += nrows;
        SG_CUDA(cudaEventRecord(hp->ev_in[c], hp->s_in));
        goto issued;
      }
      if (gather) {  // GPU gather of the chunk's referenced rows from the mapped user array
        // two gather streams: chunk c+1's gather starts while chunk c's last CTAs drain, so
        // the link does not idle at every chunk boundary; the apply of chunk c waits for the
        // gathers of chunks c and c-1 (each stream is ordered, so that covers every chunk <= c)
        cudaStream_t gs = (gather_streams > 1 && (c & 1)) ? hp->s_in2 : hp->s_in;
        for (int f = 0; f < nfields; ++f) {
          if (tma_gather)
            launch_gather_tma(gsrc_host[f], s->source_nnodes, hp->pieces.as<int2>(), hp->pdst.as<int64_t>(),
                              hp->csrc[f]->as<double>(), hp->pb[c], hp->pb[c + 1], p.levels, hp->piece_rows, gs,
                              gather_ctas);
          else
            launch_gather_rows(gsrc_host[f], hp->gsrc.as<int32_t>(), hp->csrc[f]->as<double>(), hp->cb[c],
                               hp->cb[c + 1], p.levels, gs);
        }
        copied += hp->cb[c + 1] - hp->cb[c];
        SG_CUDA(cudaEventRecord(hp->ev_in[c], gs));
        if (gather_streams > 1 && c > 0) SG_CUDA(cudaStreamWaitEvent(hp->s_cmp, hp->ev_in[c - 1], 0));
        goto issued;
      }
      {
      int packed_before = 0;
      for (int q = 0; q < c; ++q) packed_before += !hp->direct[q];
      const int slot = packed_before % HostPlan::kRing;
      // slot free: the last packed chunk that used it has been copied
      for (int q = c - 1, seen = 0; q >= 0 && seen < HostPlan::kRing; --q)
        if (!hp->direct[q] && ++seen == HostPlan::kRing) SG_CUDA(cudaEventSynchronize(hp->ev_in[q]));
      const auto& runs = hp->cruns[c];
      const int64_t base = hp->cb[c], nrows = hp->cb[c + 1] - hp->cb[c];
      const int nr = (int)runs.size();
      const int grain = std::max(1, nr / (host_pool().size() * 4));
      for (int f = 0; f < nfields; ++f) {
        char* stage = static_cast<char*>(hp->ring[(size_t)f * HostPlan::kRing + slot]);
        const char* host = reinterpret_cast<const char*>(host_src[f]);
        host_pool().parallel_for((nr + grain - 1) / grain, [&](int b) {
          for (int k = b * grain; k < std::min(nr, (b + 1) * grain); ++k)
            copy_rows_nt(stage + (runs[k].dst - base) * row, host + runs[k].src * row, (size_t)runs[k].len * row);
          _mm_sfence();
        });
        if (nrows)
          SG_CUDA(cudaMemcpyAsync(hp->csrc[f]->as<char>() + base * row, stage, (size_t)nrows * row,
                                  cudaMemcpyHostToDevice, hp->s_in));
      }
      copied += nrows;
      }
    } else {
      for (int f = 0; f < nfields; ++f) {
        char* dev = p.src[f]->buf.as<char>();
        const char* host = reinterpret_cast<const char*>(host_src[f]);
        for (auto& r : hp->runs[c])
          SG_CUDA(cudaMemcpyAsync(dev + r.first * row, host + r.first * row, (size_t)(r.second - r.first) * row,
                                  cudaMemcpyHostToDevice, hp->s_in));
      }
    }
    SG_CUDA(cudaEventRecord(hp->ev_in[c], hp->s_in));
  issued:
    SG_CUDA(cudaStreamWaitEvent(hp->s_cmp, hp->ev_in[c], 0));
    const int64_t te = hp->t_end[c];
    for (int f0 = 0; f0 < nfields; f0 += kMaxFields) {
      ApplyArgs a = make_args(s, p, f0, tprev, te);
      if (compact) {
        a.idx = hp->cidx.as<int4>();
        for (int f = 0; f < a.nfields; ++f) {
          a.src[f] = hp->csrc[f0 + f]->as<double>();
          a.src_pitch[f] = p.levels;
        }
      }
      launch_apply(a, variant, hp->s_cmp);
    }
    SG_CUDA(cudaEventRecord(hp->ev_cmp[c], hp->s_cmp));
    SG_CUDA(cudaStreamWaitEvent(hp->s_out, hp->ev_cmp[c], 0));
    if (te > tprev)
      for (int f = 0; f < nfields; ++f)
        SG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(host_dst[f]) + tprev * row,
                                p.dst[f]->buf.as<char>() + tprev * row, (size_t)(te - tprev) * row,
                                cudaMemcpyDeviceToHost, hp->s_out));
    tprev = te;
  }
  SG_CUDA(cudaStreamSynchronize(hp->s_out));
  SG_CUDA(cudaStreamSynchronize(hp->s_cmp));
  SG_CUDA(cudaStreamSynchronize(hp->s_in));
  SG_CUDA(cudaStreamSynchronize(hp->s_in2));
  if (out_rows_copied) *out_rows_copied = compact ? copied : hp->rows_copied;
  SG_API_END
}

}  // extern "C"
