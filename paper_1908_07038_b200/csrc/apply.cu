// apply_remap on the device (interp.py:206-228): a multi-level, multi-field 3-point gather
// SpMM.  Memory-bound (≈0.16 flop/B); no tensor cores.
//
//   dst[t, l] = (w0*src[n0, l] + w1*src[n1, l]) + w2*src[n2, l]
//
// rounded exactly like numpy's evaluation of interp.py:219-223 (three separately rounded
// products, two separately rounded adds: __dmul_rn / __dadd_rn are never FMA-contracted).
//
// Kernels (all take a target range [t0, t1) so a host pipeline can run chunks):
//  * warp per target (default).  Lanes span the level dimension; every lane issues all of
//    its 3 x ITERS row loads before the arithmetic (9-15 independent loads in flight per
//    lane).  16-B loads when rows are 16-B aligned (even pitch), 8-B loads otherwise (dense
//    137-level rows).  Source rows have no reuse (U/m ≈ 3.0): loads bypass
//    L1 (ld.global.nc.L1::no_allocate), stores stream (st.global.cs).
//  * TMA bulk (variant 2): a producer warp issues cp.async.bulk global->shared copies of the
//    3 rows of each target of a tile (16-B aligned superset of every row, so any pitch
//    works) into a STAGES-deep ring guarded by full/empty mbarriers; 8 consumer warps (one
//    target each) compute from shared memory and stream the rows out.
//  * thread per target for levels <= 8.
// The host-buffer pipeline (sg_remap_execute_host) lives in execute_host.cu.
#include <algorithm>
#include <mutex>
#include <vector>

#include "apply_internal.cuh"
#include "tma.cuh"

namespace sg {
namespace {
using detail::ApplyArgs;
using detail::kMaxFields;
using namespace tma;



__device__ __forceinline__ double2 ldg_stream2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg_stream1(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// HINT: L2 prefetch size qualifier (0 none, 1 128B, 2 256B)
template <int HINT>
__device__ __forceinline__ double ldg_hint(const double* p) {
  double v;
  if (HINT == 2)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if (HINT == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double4 ldg_w4(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ double combine(double w0, double w1, double w2, double a, double b, double c) {
  // numpy: (w0*a + w1*b) + w2*c, each op rounded (interp.py:219-223)
  return __dadd_rn(__dadd_rn(__dmul_rn(w0, a), __dmul_rn(w1, b)), __dmul_rn(w2, c));
}
// 4-point stencils (structured bilinear): ((w0*a + w1*b) + w2*c) + w3*d, left to right
__device__ __forceinline__ double combine4(double4 w, double a, double b, double c, double d) {
  return __dadd_rn(combine(w.x, w.y, w.z, a, b, c), __dmul_rn(w.w, d));
}

// ---- warp per target, 16-B loads (even pitch) ------------------------------------------------
template <int ITERS>
__global__ void __launch_bounds__(256) apply_warp_v2(ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t pos = a.t0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (pos >= a.t1) return;
  const int64_t t = a.list ? (int64_t)__ldg(a.list + pos) : pos;
  const int4 id = __ldg(a.idx + t);
  const double4 wt = ldg_w4(a.w + t);
  const int nvec = (a.levels + 1) >> 1;  // even pitch: the pad element of an odd row exists
  const bool odd = a.levels & 1;
  for (int f = 0; f < a.nfields; ++f) {
    const double2* r0 = reinterpret_cast<const double2*>(a.src[f] + (int64_t)id.x * a.src_pitch[f]);
    const double2* r1 = reinterpret_cast<const double2*>(a.src[f] + (int64_t)id.y * a.src_pitch[f]);
    const double2* r2 = reinterpret_cast<const double2*>(a.src[f] + (int64_t)id.z * a.src_pitch[f]);
    double* outp = a.dst[f] + t * a.dst_pitch[f];
    double2 v0[ITERS], v1[ITERS], v2[ITERS];
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const int k = lane + 32 * i;
      if (k < nvec) {
        v0[i] = ldg_stream2(r0 + k);
        v1[i] = ldg_stream2(r1 + k);
        v2[i] = ldg_stream2(r2 + k);
      }
    }
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const int k = lane + 32 * i;
      if (k < nvec) {
        double2 o;
        o.x = combine(wt.x, wt.y, wt.z, v0[i].x, v1[i].x, v2[i].x);
        o.y = combine(wt.x, wt.y, wt.z, v0[i].y, v1[i].y, v2[i].y);
        if (odd && k == nvec - 1)
          __stcs(outp + 2 * k, o.x);  // never touch the next row
        else
          __stcs(reinterpret_cast<double2*>(outp) + k, o);
      }
    }
  }
}

// ---- warp per target, 8-B loads (any pitch; dense odd rows) ----------------------------------
// SPLIT: one warp per (target, field) instead of per target — F fields sharing one stencil then
// keep as many gathers in flight as one field does (a warp looping over F fields waits F
// latencies); the stencil entry is re-read per field from L1/L2.
template <int ITERS, int HINT = 0, bool SPLIT = false>
__global__ void __launch_bounds__(256) apply_warp_v1(ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t pos = a.t0 + (SPLIT ? wg / a.nfields : wg);
  if (pos >= a.t1) return;
  const int f_lo = SPLIT ? (int)(wg % a.nfields) : 0, f_hi = SPLIT ? f_lo + 1 : a.nfields;
  const int64_t t = a.list ? (int64_t)__ldg(a.list + pos) : pos;
  const int4 id = __ldg(a.idx + t);
  const double4 wt = ldg_w4(a.w + t);
  const int L = a.levels;
  for (int f = f_lo; f < f_hi; ++f) {
    const double* r0 = a.src[f] + (int64_t)id.x * a.src_pitch[f];
    const double* r1 = a.src[f] + (int64_t)id.y * a.src_pitch[f];
    const double* r2 = a.src[f] + (int64_t)id.z * a.src_pitch[f];
    double* outp = a.dst[f] + t * a.dst_pitch[f];
    double v0[ITERS], v1[ITERS], v2[ITERS];
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const int k = lane + 32 * i;
      if (k < L) {
        v0[i] = ldg_hint<HINT>(r0 + k);
        v1[i] = ldg_hint<HINT>(r1 + k);
        v2[i] = ldg_hint<HINT>(r2 + k);
      }
    }
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const int k = lane + 32 * i;
      if (k < L) __stcs(outp + k, combine(wt.x, wt.y, wt.z, v0[i], v1[i], v2[i]));
    }
  }
}

// ---- 4-point stencils (structured bilinear, bilinear.cu): warp per target, 8-B loads -------
template <int ITERS>
__global__ void __launch_bounds__(256) apply4_warp(ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t pos = a.t0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (pos >= a.t1) return;
  const int64_t t = a.list ? (int64_t)__ldg(a.list + pos) : pos;
  const int4 id = __ldg(a.idx + t);
  const double4 wt = ldg_w4(a.w + t);
  const int L = a.levels;
  for (int f = 0; f < a.nfields; ++f) {
    const double* r0 = a.src[f] + (int64_t)id.x * a.src_pitch[f];
    const double* r1 = a.src[f] + (int64_t)id.y * a.src_pitch[f];
    const double* r2 = a.src[f] + (int64_t)id.z * a.src_pitch[f];
    const double* r3 = a.src[f] + (int64_t)id.w * a.src_pitch[f];
    double* outp = a.dst[f] + t * a.dst_pitch[f];
    if (ITERS > 0) {
      double v0[ITERS > 0 ? ITERS : 1], v1[ITERS > 0 ? ITERS : 1], v2[ITERS > 0 ? ITERS : 1], v3[ITERS > 0 ? ITERS : 1];
#pragma unroll
      for (int i = 0; i < ITERS; ++i) {
        const int k = lane + 32 * i;
        if (k < L) {
          v0[i] = ldg_stream1(r0 + k);
          v1[i] = ldg_stream1(r1 + k);
          v2[i] = ldg_stream1(r2 + k);
          v3[i] = ldg_stream1(r3 + k);
        }
      }
#pragma unroll
      for (int i = 0; i < ITERS; ++i) {
        const int k = lane + 32 * i;
        if (k < L) __stcs(outp + k, combine4(wt, v0[i], v1[i], v2[i], v3[i]));
      }
    } else {
      for (int l = lane; l < L; l += 32)
        __stcs(outp + l, combine4(wt, ldg_stream1(r0 + l), ldg_stream1(r1 + l), ldg_stream1(r2 + l), ldg_stream1(r3 + l)));
    }
  }
}

// Any number of levels (> 256): looped.
__global__ void __launch_bounds__(256) apply_warp_loop(ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t pos = a.t0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (pos >= a.t1) return;
  const int64_t t = a.list ? (int64_t)__ldg(a.list + pos) : pos;
  const int4 id = __ldg(a.idx + t);
  const double4 wt = ldg_w4(a.w + t);
  for (int f = 0; f < a.nfields; ++f) {
    const double* r0 = a.src[f] + (int64_t)id.x * a.src_pitch[f];
    const double* r1 = a.src[f] + (int64_t)id.y * a.src_pitch[f];
    const double* r2 = a.src[f] + (int64_t)id.z * a.src_pitch[f];
    double* outp = a.dst[f] + t * a.dst_pitch[f];
    for (int l = lane; l < a.levels; l += 32)
      __stcs(outp + l, combine(wt.x, wt.y, wt.z, ldg_stream1(r0 + l), ldg_stream1(r1 + l), ldg_stream1(r2 + l)));
  }
}

// Thread per target for few levels (levels <= 8): the stencil loads of a warp coalesce.
__global__ void __launch_bounds__(256) apply_thread_short(ApplyArgs a) {
  const int64_t pos = a.t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= a.t1) return;
  const int64_t t = a.list ? (int64_t)__ldg(a.list + pos) : pos;
  const int4 id = __ldg(a.idx + t);
  const double4 wt = ldg_w4(a.w + t);
  for (int f = 0; f < a.nfields; ++f) {
    const double* r0 = a.src[f] + (int64_t)id.x * a.src_pitch[f];
    const double* r1 = a.src[f] + (int64_t)id.y * a.src_pitch[f];
    const double* r2 = a.src[f] + (int64_t)id.z * a.src_pitch[f];
    double* outp = a.dst[f] + t * a.dst_pitch[f];
    for (int l = 0; l < a.levels; ++l)
      outp[l] = combine(wt.x, wt.y, wt.z, __ldg(r0 + l), __ldg(r1 + l), __ldg(r2 + l));
  }
}

// ---- TMA bulk-copy staged gather ---------------------------------------------------------------

// mbarrier / bulk-copy helpers: tma.cuh

// smem: ring of `stages` stages x 3*TILE row slots of `slot` doubles; each slot holds the
// 16-B aligned superset of one source row (the row starts at element off = addr%16/8).
// Producer warp (lanes = targets of the tile) prefetches the NEXT tile's stencil entries
// while the current copies fly, so the index load is off the critical path; consumer warps
// load their weights before waiting on the tile's full barrier.
template <int TILE>
__global__ void __launch_bounds__((TILE + 1) * 32) apply_bulk(ApplyArgs a, int slot, int stages) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + stages;
  unsigned char* offs = reinterpret_cast<unsigned char*>(empty + stages);  // [stages][3*TILE]
  double* ring = reinterpret_cast<double*>(smem_raw + ((16 * stages + 3 * TILE * stages + 127) / 128) * 128);
  const int64_t ntiles = (a.t1 - a.t0 + TILE - 1) / TILE;
  const int64_t nwork = ntiles * a.nfields;  // work item = (tile, field)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TILE);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == TILE) {
    // ===== producer warp =====
    int4 next_id = make_int4(0, 0, 0, 0);
    {
      const int64_t item = blockIdx.x;
      if (item < nwork) {
        const int64_t tb = a.t0 + (item / a.nfields) * TILE;
        if (lane < TILE && tb + lane < a.t1) next_id = __ldg(a.idx + tb + lane);
      }
    }
    int it = 0;
    for (int64_t item = blockIdx.x; item < nwork; item += gridDim.x, ++it) {
      const int stage = it % stages;
      const int4 id = next_id;
      {  // prefetch the next item's stencil entries
        const int64_t nitem = item + gridDim.x;
        if (nitem < nwork) {
          const int64_t ntb = a.t0 + (nitem / a.nfields) * TILE;
          if (lane < TILE && ntb + lane < a.t1) next_id = __ldg(a.idx + ntb + lane);
        }
      }
      if (it >= stages) mbar_wait(&empty[stage], ((it / stages) - 1) & 1);
      const int64_t tile = item / a.nfields;
      const int f = (int)(item % a.nfields);
      const int64_t tb = a.t0 + tile * TILE;
      const int nt = (int)min((int64_t)TILE, a.t1 - tb);
      uint32_t bytes[3] = {0, 0, 0};
      const double* rows[3] = {nullptr, nullptr, nullptr};
      if (lane < nt) {
        const int ids[3] = {id.x, id.y, id.z};
        for (int c = 0; c < 3; ++c) {
          const double* r = a.src[f] + (int64_t)ids[c] * a.src_pitch[f];
          const uintptr_t p = reinterpret_cast<uintptr_t>(r);
          const uintptr_t s0 = p & ~uintptr_t(15), s1 = (p + (uintptr_t)a.levels * 8 + 15) & ~uintptr_t(15);
          rows[c] = reinterpret_cast<const double*>(s0);
          bytes[c] = (uint32_t)(s1 - s0);
          offs[stage * 3 * TILE + 3 * lane + c] = (unsigned char)((p - s0) >> 3);
        }
      }
      uint32_t total = bytes[0] + bytes[1] + bytes[2];
      for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
      if (lane == 0) mbar_expect_tx(&full[stage], total);
      __syncwarp();
      if (lane < nt) {
        double* base = ring + (size_t)stage * 3 * TILE * slot;
        for (int c = 0; c < 3; ++c) bulk_g2s(base + (3 * lane + c) * slot, rows[c], bytes[c], &full[stage]);
      }
    }
    return;
  }
  // ===== consumer warps: warp j computes target j of the tile =====
  int it = 0;
  for (int64_t item = blockIdx.x; item < nwork; item += gridDim.x, ++it) {
    const int stage = it % stages;
    const int64_t tile = item / a.nfields;
    const int f = (int)(item % a.nfields);
    const int64_t tb = a.t0 + tile * TILE;
    const int nt = (int)min((int64_t)TILE, a.t1 - tb);
    double4 wt = make_double4(0, 0, 0, 0);
    if (warp < nt) wt = ldg_w4(a.w + tb + warp);
    mbar_wait(&full[stage], (it / stages) & 1);
    if (warp < nt) {
      const int64_t t = tb + warp;
      const double* base = ring + (size_t)stage * 3 * TILE * slot;
      const unsigned char* o = offs + stage * 3 * TILE + 3 * warp;
      const double* r0 = base + (3 * warp + 0) * slot + o[0];
      const double* r1 = base + (3 * warp + 1) * slot + o[1];
      const double* r2 = base + (3 * warp + 2) * slot + o[2];
      double* outp = a.dst[f] + t * a.dst_pitch[f];
      for (int l = lane; l < a.levels; l += 32) __stcs(outp + l, combine(wt.x, wt.y, wt.z, r0[l], r1[l], r2[l]));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
  }
}

template <int TILE>
void launch_bulk(ApplyArgs a, int L, int64_t m, size_t budget, cudaStream_t st);

__global__ void mark_sources(const int4* idx, int64_t m, int k, unsigned char* mark) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int4 id = idx[t];
  mark[id.x] = 1;
  mark[id.y] = 1;
  mark[id.z] = 1;
  if (k == 4) mark[id.w] = 1;
}

__global__ void count_marks(const unsigned char* mark, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += mark[i];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

__global__ void pack_stencil(const int32_t* idxk, const double* wk, int64_t m, int k, int4* idx, double4* w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int32_t* i = idxk + k * t;
  const double* x = wk + k * t;
  idx[t] = make_int4(i[0], i[1], i[2], k == 4 ? i[3] : 0);
  w[t] = make_double4(x[0], x[1], x[2], k == 4 ? x[3] : 0.0);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int TILE>
void launch_bulk(ApplyArgs a, int L, int64_t m, size_t budget, cudaStream_t st) {
  const int slot = ((L + 2) * 8 + 15) / 16 * 2;  // doubles; holds the 16-B aligned superset
  const size_t stage_bytes = (size_t)3 * TILE * slot * 8;
  const int stages = (int)std::min<size_t>(8, std::max<size_t>(2, budget / stage_bytes));
  const size_t hdr = ((16 * stages + 3 * TILE * stages + 127) / 128) * 128;
  const size_t smem = hdr + stages * stage_bytes;
  SG_REQUIRE(smem <= 220 * 1024, "levels too large for the bulk-copy variant");
  SG_CUDA(cudaFuncSetAttribute(apply_bulk<TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, apply_bulk<TILE>, (TILE + 1) * 32, smem));
  const int64_t nwork = (m + TILE - 1) / TILE * a.nfields;
  const int64_t grid = std::min<int64_t>((int64_t)num_sms() * std::max(per_sm, 1), nwork);
  apply_bulk<TILE><<<(unsigned)grid, (TILE + 1) * 32, smem, st>>>(a, slot, stages);
}

// Launches the apply of targets [t0, t1) for up to kMaxFields field pairs.
}  // namespace

namespace detail {
// Threads per block of the warp-per-target kernels: 2 warps (targets).  Register use caps a
// SM at 32 resident warps either way; small blocks retire and refill at target granularity
// instead of waiting for the slowest of 8 gathers (cfg3: 1.085 vs 1.096 ms with 8-warp blocks,
// profiles/r01_apply_variant_sweep2.jsonl).  Variant 16 keeps 8-warp blocks for comparison.
static int warp_block_threads(int variant) { return variant == 16 ? 256 : 64; }

void launch_apply(ApplyArgs a, int variant, cudaStream_t st) {
  const int64_t m = a.t1 - a.t0;
  if (m <= 0) return;
  const int L = a.levels;
  if (a.k == 4) {
    const int tpb = warp_block_threads(variant);
    const unsigned grid = (unsigned)((m * 32 + tpb - 1) / tpb);
    switch ((L + 31) / 32) {
      case 1: apply4_warp<1><<<grid, tpb, 0, st>>>(a); break;
      case 2: apply4_warp<2><<<grid, tpb, 0, st>>>(a); break;
      case 3: apply4_warp<3><<<grid, tpb, 0, st>>>(a); break;
      case 4: apply4_warp<4><<<grid, tpb, 0, st>>>(a); break;
      case 5: apply4_warp<5><<<grid, tpb, 0, st>>>(a); break;
      case 6: apply4_warp<6><<<grid, tpb, 0, st>>>(a); break;
      default: apply4_warp<0><<<grid, tpb, 0, st>>>(a); break;
    }
    SG_CUDA_LAUNCH();
    return;
  }
  bool even = true;
  for (int f = 0; f < a.nfields; ++f) even = even && a.src_pitch[f] % 2 == 0 && a.dst_pitch[f] % 2 == 0;
  if ((variant == 2 || variant == 6 || variant == 7) && L >= 2 && a.k == 3 && !a.list) {
    if (variant == 2) launch_bulk<4>(a, L, m, 42 * 1024, st);       // 3 stages, ~5 CTAs/SM
    else if (variant == 6) launch_bulk<4>(a, L, m, 56 * 1024, st);  // 4 stages, ~4 CTAs/SM
    else launch_bulk<2>(a, L, m, 21 * 1024, st);                    // 3 stages, ~10 CTAs/SM
  } else if (L <= 8) {
    apply_thread_short<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(a);
  } else {
    const int tpb = warp_block_threads(variant);  // warp per target
    const unsigned grid = (unsigned)((m * 32 + tpb - 1) / tpb);
    const int nv = (L + 1) / 2;
    if (even && variant != 3) {
      switch (nv <= 32 ? 1 : nv <= 64 ? 2 : nv <= 96 ? 3 : nv <= 128 ? 4 : 0) {
        case 1: apply_warp_v2<1><<<grid, tpb, 0, st>>>(a); break;
        case 2: apply_warp_v2<2><<<grid, tpb, 0, st>>>(a); break;
        case 3: apply_warp_v2<3><<<grid, tpb, 0, st>>>(a); break;
        case 4: apply_warp_v2<4><<<grid, tpb, 0, st>>>(a); break;
        default: apply_warp_loop<<<grid, tpb, 0, st>>>(a); break;
      }
    } else if ((variant == 4 || variant == 5) && (L + 31) / 32 == 5) {
      if (variant == 4) apply_warp_v1<5, 2><<<grid, tpb, 0, st>>>(a);  // L2::256B prefetch
      else apply_warp_v1<5, 1><<<grid, tpb, 0, st>>>(a);                // L2::128B prefetch
    } else if (a.nfields > 1 && (L + 31) / 32 <= 5) {  // F fields: a warp per (target, field)
      const unsigned gridf = (unsigned)((m * a.nfields * 32 + tpb - 1) / tpb);
      switch ((L + 31) / 32) {
        case 1: apply_warp_v1<1, 0, true><<<gridf, tpb, 0, st>>>(a); break;
        case 2: apply_warp_v1<2, 0, true><<<gridf, tpb, 0, st>>>(a); break;
        case 3: apply_warp_v1<3, 0, true><<<gridf, tpb, 0, st>>>(a); break;
        case 4: apply_warp_v1<4, 0, true><<<gridf, tpb, 0, st>>>(a); break;
        default: apply_warp_v1<5, 0, true><<<gridf, tpb, 0, st>>>(a); break;
      }
    } else {
      switch ((L + 31) / 32) {
        case 1: apply_warp_v1<1><<<grid, tpb, 0, st>>>(a); break;
        case 2: apply_warp_v1<2><<<grid, tpb, 0, st>>>(a); break;
        case 3: apply_warp_v1<3><<<grid, tpb, 0, st>>>(a); break;
        case 4: apply_warp_v1<4><<<grid, tpb, 0, st>>>(a); break;
        case 5: apply_warp_v1<5><<<grid, tpb, 0, st>>>(a); break;
        case 6: apply_warp_v1<6><<<grid, tpb, 0, st>>>(a); break;
        case 7: apply_warp_v1<7><<<grid, tpb, 0, st>>>(a); break;
        case 8: apply_warp_v1<8><<<grid, tpb, 0, st>>>(a); break;
        default: apply_warp_loop<<<grid, tpb, 0, st>>>(a); break;
      }
    }
  }
  SG_CUDA_LAUNCH();
}



FieldPairs check_pairs(const Stencil* s, const uint64_t* src_fields, const uint64_t* dst_fields, int nfields) {
  SG_REQUIRE(nfields >= 1, "nfields must be >= 1");
  SG_REQUIRE(src_fields && dst_fields, "null field arrays");
  FieldPairs p;
  p.src.resize(nfields);
  p.dst.resize(nfields);
  for (int f = 0; f < nfields; ++f) {
    Field* a = p.src[f] = get<Field>(src_fields[f], ObjKind::Field);
    Field* b = p.dst[f] = get<Field>(dst_fields[f], ObjKind::Field);
    // exact reference messages, interp.py:208-217
    if (a->npts != s->source_nnodes)
      throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: source field has %lld points, weights expect %lld",
                  (long long)a->npts, (long long)s->source_nnodes);
    if (b->npts != s->m)
      throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: target field has %lld points, weights cover %lld",
                  (long long)b->npts, (long long)s->m);
    if (a->levels != b->levels) throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: level counts differ");
    SG_REQUIRE(a->itemsize == 8 && b->itemsize == 8, "apply_remap on device needs real64 fields");
    SG_REQUIRE(a->device == s->device && b->device == s->device, "fields and stencil live on different devices");
    if (p.levels < 0) p.levels = a->levels;
    SG_REQUIRE(a->levels == p.levels, "all field pairs of one call must have equal levels");
  }
  return p;
}

ApplyArgs make_args(const Stencil* s, const FieldPairs& p, int f0, int64_t t0, int64_t t1) {
  ApplyArgs a{};
  a.idx = s->idx.as<int4>();
  a.w = s->w.as<double4>();
  a.t0 = t0;
  a.t1 = t1;
  a.k = s->k;
  a.levels = p.levels;
  a.nfields = std::min<int>(kMaxFields, (int)p.src.size() - f0);
  for (int f = 0; f < a.nfields; ++f) {
    a.src[f] = p.src[f0 + f]->buf.as<double>();
    a.dst[f] = p.dst[f0 + f]->buf.as<double>();
    a.src_pitch[f] = p.src[f0 + f]->pitch;
    a.dst_pitch[f] = p.dst[f0 + f]->pitch;
  }
  return a;
}

// ---- host pipeline plan (per stencil, built on first use) -----------------------------------
}  // namespace detail

void stencil_finalize(Stencil* s, const int32_t* d_idx3, const double* d_w3, cudaStream_t st) {
  s->idx.alloc(s->device, (size_t)std::max<int64_t>(s->m, 1) * sizeof(int4));
  s->w.alloc(s->device, (size_t)std::max<int64_t>(s->m, 1) * sizeof(double4));
  if (s->m > 0) {
    pack_stencil<<<(unsigned)((s->m + 255) / 256), 256, 0, st>>>(d_idx3, d_w3, s->m, s->k, s->idx.as<int4>(),
                                                                 s->w.as<double4>());
    SG_CUDA_LAUNCH();
  }
  DevBuf mark, cnt;
  mark.alloc(s->device, (size_t)std::max<int64_t>(s->source_nnodes, 1));
  cnt.alloc(s->device, sizeof(unsigned long long));
  SG_CUDA(cudaMemsetAsync(mark.ptr, 0, mark.bytes, st));
  SG_CUDA(cudaMemsetAsync(cnt.ptr, 0, cnt.bytes, st));
  if (s->m > 0) {
    mark_sources<<<(unsigned)((s->m + 255) / 256), 256, 0, st>>>(s->idx.as<int4>(), s->m, s->k,
                                                                 mark.as<unsigned char>());
    SG_CUDA_LAUNCH();
    count_marks<<<1024, 256, 0, st>>>(mark.as<unsigned char>(), s->source_nnodes, cnt.as<unsigned long long>());
    SG_CUDA_LAUNCH();
  }
  unsigned long long u = 0;
  SG_CUDA(cudaMemcpyAsync(&u, cnt.ptr, sizeof(u), cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  s->distinct_sources = (int64_t)u;
}

}  // namespace sg

using namespace sg;
using namespace sg::detail;

extern "C" {

int32_t sg_stencil_create_k(int32_t device, const int64_t* nodes, const double* weights, int64_t m, int32_t k,
                            int64_t source_nnodes, uint64_t* out_stencil) {
  SG_API_BEGIN
  SG_REQUIRE(out_stencil, "null out pointer");
  SG_REQUIRE(k == 3 || k == 4, "stencils have 3 or 4 points, got %d", k);
  SG_REQUIRE(m >= 0 && source_nnodes >= 0, "negative size");
  SG_REQUIRE(m == 0 || (nodes && weights), "null stencil arrays");
  SG_REQUIRE(source_nnodes < (int64_t)INT32_MAX, "source mesh too large for int32 indices");
  std::vector<int32_t> idxk((size_t)m * k);
  for (int64_t i = 0; i < m * k; ++i) {
    SG_REQUIRE(nodes[i] >= 0 && nodes[i] < source_nnodes, "stencil node %lld out of range [0, %lld)",
               (long long)nodes[i], (long long)source_nnodes);
    idxk[i] = (int32_t)nodes[i];
  }
  DeviceScope ds(device);
  auto s = std::make_unique<Stencil>();
  s->device = device;
  s->m = m;
  s->k = k;
  s->source_nnodes = source_nnodes;
  DevBuf di, dw;
  di.alloc(device, std::max<size_t>(idxk.size(), 1) * sizeof(int32_t));
  dw.alloc(device, std::max<size_t>((size_t)m * k, 1) * sizeof(double));
  if (m) {
    SG_CUDA(cudaMemcpy(di.ptr, idxk.data(), idxk.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    SG_CUDA(cudaMemcpy(dw.ptr, weights, (size_t)m * k * sizeof(double), cudaMemcpyHostToDevice));
  }
  stencil_finalize(s.get(), di.as<int32_t>(), dw.as<double>(), 0);
  *out_stencil = registry_put(s.release());
  SG_API_END
}

int32_t sg_stencil_create(int32_t device, const int64_t* nodes, const double* weights, int64_t m,
                          int64_t source_nnodes, uint64_t* out_stencil) {
  return sg_stencil_create_k(device, nodes, weights, m, 3, source_nnodes, out_stencil);
}

int32_t sg_stencil_info(uint64_t stencil, int64_t* out_m, int64_t* out_source_nnodes,
                        int64_t* out_distinct_sources) {
  SG_API_BEGIN
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  if (out_m) *out_m = s->m;
  if (out_source_nnodes) *out_source_nnodes = s->source_nnodes;
  if (out_distinct_sources) *out_distinct_sources = s->distinct_sources;
  SG_API_END
}

int32_t sg_remap_apply(uint64_t stencil, const uint64_t* src_fields, const uint64_t* dst_fields, int32_t nfields,
                       int32_t variant, uint64_t stream) {
  SG_API_BEGIN
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  FieldPairs p = check_pairs(s, src_fields, dst_fields, nfields);
  DeviceScope ds(s->device);
  for (int f0 = 0; f0 < nfields; f0 += kMaxFields) launch_apply(make_args(s, p, f0, 0, s->m), variant, as_stream(stream));
  SG_API_END
}

int32_t sg_remap_apply_range(uint64_t stencil, const uint64_t* src_fields, const uint64_t* dst_fields,
                             int32_t nfields, int64_t t0, int64_t t1, int32_t variant, uint64_t stream) {
  SG_API_BEGIN
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  FieldPairs p = check_pairs(s, src_fields, dst_fields, nfields);
  SG_REQUIRE(0 <= t0 && t0 <= t1 && t1 <= s->m, "target range [%lld, %lld) outside [0, %lld)", (long long)t0,
             (long long)t1, (long long)s->m);
  DeviceScope ds(s->device);
  for (int f0 = 0; f0 < nfields; f0 += kMaxFields) launch_apply(make_args(s, p, f0, t0, t1), variant, as_stream(stream));
  SG_API_END
}

int32_t sg_remap_apply_list(uint64_t stencil, const uint64_t* src_fields, const uint64_t* dst_fields,
                            int32_t nfields, const int32_t* dev_targets, int64_t count, int32_t variant,
                            uint64_t stream) {
  SG_API_BEGIN
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  FieldPairs p = check_pairs(s, src_fields, dst_fields, nfields);
  SG_REQUIRE(count >= 0 && (count == 0 || dev_targets), "bad target list");
  DeviceScope ds(s->device);
  for (int f0 = 0; f0 < nfields; f0 += kMaxFields) {
    ApplyArgs a = make_args(s, p, f0, 0, count);
    a.list = dev_targets;
    launch_apply(a, variant, as_stream(stream));
  }
  SG_API_END
}

}  // extern "C"
