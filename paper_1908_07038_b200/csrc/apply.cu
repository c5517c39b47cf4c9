// apply_remap on the device (interp.py:206-228): a multi-level, multi-field 3-point gather
// SpMM.  Memory-bound (≈0.16 flop/B); no tensor cores.
//
//   dst[t, l] = (w0*src[n0, l] + w1*src[n1, l]) + w2*src[n2, l]
//
// rounded exactly like numpy's evaluation of interp.py:219-223 (three separately rounded
// products, two separately rounded adds: __dmul_rn / __dadd_rn are never FMA-contracted).
//
// Two kernels:
//  * variant 1 (default): one warp per target row.  Lanes span the level dimension with
//    16-B (double2) loads; every lane issues all of its 3 x ITERS row loads before the
//    arithmetic so ~9 independent 16-B requests per lane are in flight.  Source rows have
//    no reuse (U/m ≈ 3.0), so loads bypass L1 (ld.global.nc.L1::no_allocate)
//    and stores stream (st.global.cs).
//  * variant 2: TMA bulk copies.  A persistent CTA per SM slot walks tiles of TILE targets;
//    one elected thread issues cp.async.bulk (global -> shared, mbarrier complete_tx) for
//    the 3*TILE referenced source rows of a tile into a STAGES-deep ring, the CTA computes
//    from shared memory and streams the rows out.
#include <algorithm>
#include <vector>

#include "stencil.cuh"

namespace sg {
namespace {

constexpr int kMaxFields = 8;

struct ApplyArgs {
  const int4* idx;
  const double4* w;
  int64_t m;
  int32_t levels;
  int32_t nfields;
  const double* src[kMaxFields];
  double* dst[kMaxFields];
  int64_t src_pitch[kMaxFields];
  int64_t dst_pitch[kMaxFields];
};

__device__ __forceinline__ double2 ldg_stream2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg_stream1(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ double4 ldg_w4(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ double combine(double w0, double w1, double w2, double a, double b,
                                          double c) {
  // numpy: (w0*a + w1*b) + w2*c, each op rounded (interp.py:219-223)
  return __dadd_rn(__dadd_rn(__dmul_rn(w0, a), __dmul_rn(w1, b)), __dmul_rn(w2, c));
}

// ---- variant 1: warp per target, 16-B vector loads over levels --------------------------
template <int ITERS>
__global__ void __launch_bounds__(256) apply_warp_v2(ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= a.m) return;
  const int4 id = __ldg(a.idx + t);
  const double4 wt = ldg_w4(a.w + t);
  const int nvec = (a.levels + 1) >> 1;  // pitch is even, padding is zero
  for (int f = 0; f < a.nfields; ++f) {
    const double2* r0 = reinterpret_cast<const double2*>(a.src[f] + (int64_t)id.x * a.src_pitch[f]);
    const double2* r1 = reinterpret_cast<const double2*>(a.src[f] + (int64_t)id.y * a.src_pitch[f]);
    const double2* r2 = reinterpret_cast<const double2*>(a.src[f] + (int64_t)id.z * a.src_pitch[f]);
    double2* out = reinterpret_cast<double2*>(a.dst[f] + t * a.dst_pitch[f]);
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
        __stcs(out + k, o);
      }
    }
  }
}

// Generic fallback: any pitch (odd, e.g. levels == 1), scalar loads, looped over levels.
__global__ void __launch_bounds__(256) apply_warp_scalar(ApplyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= a.m) return;
  const int4 id = __ldg(a.idx + t);
  const double4 wt = ldg_w4(a.w + t);
  for (int f = 0; f < a.nfields; ++f) {
    const double* r0 = a.src[f] + (int64_t)id.x * a.src_pitch[f];
    const double* r1 = a.src[f] + (int64_t)id.y * a.src_pitch[f];
    const double* r2 = a.src[f] + (int64_t)id.z * a.src_pitch[f];
    double* out = a.dst[f] + t * a.dst_pitch[f];
    for (int l = lane; l < a.levels; l += 32)
      __stcs(out + l, combine(wt.x, wt.y, wt.z, ldg_stream1(r0 + l), ldg_stream1(r1 + l),
                              ldg_stream1(r2 + l)));
  }
}

// Thread-per-target variant for few levels (levels <= 8): a warp covers 32 targets, so the
// stencil loads coalesce and each lane walks its target's short rows.
__global__ void __launch_bounds__(256) apply_thread_short(ApplyArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.m) return;
  const int4 id = __ldg(a.idx + t);
  const double4 wt = ldg_w4(a.w + t);
  for (int f = 0; f < a.nfields; ++f) {
    const double* r0 = a.src[f] + (int64_t)id.x * a.src_pitch[f];
    const double* r1 = a.src[f] + (int64_t)id.y * a.src_pitch[f];
    const double* r2 = a.src[f] + (int64_t)id.z * a.src_pitch[f];
    double* out = a.dst[f] + t * a.dst_pitch[f];
    for (int l = 0; l < a.levels; ++l)
      out[l] = combine(wt.x, wt.y, wt.z, __ldg(r0 + l), __ldg(r1 + l), __ldg(r2 + l));
  }
}

// ---- variant 2: TMA bulk-copy staged gather ------------------------------------------------
constexpr int kTile = 8;     // targets per tile
constexpr int kStages = 4;   // ring depth
constexpr int kV2Threads = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// smem ring: [kStages][3*kTile rows][row_elems]; one work item = (tile, field)
__global__ void __launch_bounds__(kV2Threads) apply_bulk(ApplyArgs a, int row_elems,
                                                         uint32_t row_bytes) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[kStages];
  double* ring = reinterpret_cast<double*>(smem_raw);
  const size_t stage_elems = (size_t)3 * kTile * row_elems;
  const int64_t ntiles = (a.m + kTile - 1) / kTile;
  const int64_t nwork = ntiles * a.nfields;  // work item = (tile, field)
  const int64_t first = blockIdx.x;
  const int64_t stride = gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int64_t item, int stage) {
    const int64_t tile = item / a.nfields;
    const int f = (int)(item % a.nfields);
    const int64_t t0 = tile * kTile;
    const int nt = (int)(a.m - t0 < kTile ? a.m - t0 : kTile);
    mbar_expect_tx(&full_bar[stage], (uint32_t)(3 * nt) * row_bytes);
    double* base = ring + stage * stage_elems;
    for (int j = 0; j < nt; ++j) {
      const int4 id = __ldg(a.idx + t0 + j);
      bulk_g2s(base + (3 * j + 0) * row_elems, a.src[f] + (int64_t)id.x * a.src_pitch[f], row_bytes,
               &full_bar[stage]);
      bulk_g2s(base + (3 * j + 1) * row_elems, a.src[f] + (int64_t)id.y * a.src_pitch[f], row_bytes,
               &full_bar[stage]);
      bulk_g2s(base + (3 * j + 2) * row_elems, a.src[f] + (int64_t)id.z * a.src_pitch[f], row_bytes,
               &full_bar[stage]);
    }
  };

  // prologue: fill the ring
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      const int64_t item = first + s * stride;
      if (item < nwork) issue(item, s);
    }
  }
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nvec = (a.levels + 1) >> 1;
  int it = 0;
  for (int64_t item = first; item < nwork; item += stride, ++it) {
    const int stage = it % kStages;
    const uint32_t parity = (it / kStages) & 1;
    mbar_wait(&full_bar[stage], parity);
    const int64_t tile = item / a.nfields;
    const int f = (int)(item % a.nfields);
    const int64_t t0 = tile * kTile;
    const int nt = (int)(a.m - t0 < kTile ? a.m - t0 : kTile);
    const double* base = ring + stage * stage_elems;
    // warp j handles target j of the tile (kV2Threads/32 == kTile)
    if (warp < nt) {
      const double4 wt = ldg_w4(a.w + t0 + warp);
      const double2* r0 = reinterpret_cast<const double2*>(base + (3 * warp + 0) * row_elems);
      const double2* r1 = reinterpret_cast<const double2*>(base + (3 * warp + 1) * row_elems);
      const double2* r2 = reinterpret_cast<const double2*>(base + (3 * warp + 2) * row_elems);
      double2* out = reinterpret_cast<double2*>(a.dst[f] + (t0 + warp) * a.dst_pitch[f]);
      for (int k = lane; k < nvec; k += 32) {
        const double2 x = r0[k], y = r1[k], z = r2[k];
        double2 o;
        o.x = combine(wt.x, wt.y, wt.z, x.x, y.x, z.x);
        o.y = combine(wt.x, wt.y, wt.z, x.y, y.y, z.y);
        __stcs(out + k, o);
      }
    }
    __syncthreads();  // stage fully consumed
    if (threadIdx.x == 0) {
      const int64_t next = item + (int64_t)kStages * stride;
      if (next < nwork) issue(next, stage);
    }
  }
}

__global__ void mark_sources(const int4* idx, int64_t m, unsigned char* mark) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int4 id = idx[t];
  mark[id.x] = 1;
  mark[id.y] = 1;
  mark[id.z] = 1;
}

__global__ void count_marks(const unsigned char* mark, int64_t n, unsigned long long* out) {
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += mark[i];
  atomicAdd(&s, c);
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, s);
}

__global__ void pack_stencil(const int32_t* idx3, const double* w3, int64_t m, int4* idx,
                             double4* w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  idx[t] = make_int4(idx3[3 * t], idx3[3 * t + 1], idx3[3 * t + 2], 0);
  w[t] = make_double4(w3[3 * t], w3[3 * t + 1], w3[3 * t + 2], 0.0);
}

int g_num_sms = 0;

}  // namespace

void stencil_finalize(Stencil* s, const int32_t* d_idx3, const double* d_w3, cudaStream_t st) {
  s->idx.alloc(s->device, (size_t)std::max<int64_t>(s->m, 1) * sizeof(int4));
  s->w.alloc(s->device, (size_t)std::max<int64_t>(s->m, 1) * sizeof(double4));
  if (s->m > 0) {
    pack_stencil<<<(unsigned)((s->m + 255) / 256), 256, 0, st>>>(d_idx3, d_w3, s->m,
                                                                 s->idx.as<int4>(), s->w.as<double4>());
    SG_CUDA_LAUNCH();
  }
  DevBuf mark, cnt;
  mark.alloc(s->device, (size_t)std::max<int64_t>(s->source_nnodes, 1));
  cnt.alloc(s->device, sizeof(unsigned long long));
  SG_CUDA(cudaMemsetAsync(mark.ptr, 0, mark.bytes, st));
  SG_CUDA(cudaMemsetAsync(cnt.ptr, 0, cnt.bytes, st));
  if (s->m > 0) {
    mark_sources<<<(unsigned)((s->m + 255) / 256), 256, 0, st>>>(s->idx.as<int4>(), s->m,
                                                                 mark.as<unsigned char>());
    SG_CUDA_LAUNCH();
    count_marks<<<1024, 256, 0, st>>>(mark.as<unsigned char>(), s->source_nnodes,
                                      cnt.as<unsigned long long>());
    SG_CUDA_LAUNCH();
  }
  unsigned long long u = 0;
  SG_CUDA(cudaMemcpyAsync(&u, cnt.ptr, sizeof(u), cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  s->distinct_sources = (int64_t)u;
}

}  // namespace sg

using namespace sg;

extern "C" {

int32_t sg_stencil_create(int32_t device, const int64_t* nodes, const double* weights, int64_t m,
                          int64_t source_nnodes, uint64_t* out_stencil) {
  SG_API_BEGIN
  SG_REQUIRE(out_stencil, "null out pointer");
  SG_REQUIRE(m >= 0 && source_nnodes >= 0, "negative size");
  SG_REQUIRE(m == 0 || (nodes && weights), "null stencil arrays");
  SG_REQUIRE(source_nnodes < (int64_t)INT32_MAX, "source mesh too large for int32 indices");
  std::vector<int32_t> idx3((size_t)m * 3);
  for (int64_t i = 0; i < m * 3; ++i) {
    SG_REQUIRE(nodes[i] >= 0 && nodes[i] < source_nnodes, "stencil node %lld out of range [0, %lld)",
               (long long)nodes[i], (long long)source_nnodes);
    idx3[i] = (int32_t)nodes[i];
  }
  DeviceScope ds(device);
  auto s = std::make_unique<Stencil>();
  s->device = device;
  s->m = m;
  s->source_nnodes = source_nnodes;
  DevBuf di, dw;
  di.alloc(device, std::max<size_t>(idx3.size(), 1) * sizeof(int32_t));
  dw.alloc(device, std::max<size_t>((size_t)m * 3, 1) * sizeof(double));
  if (m) {
    SG_CUDA(cudaMemcpy(di.ptr, idx3.data(), idx3.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    SG_CUDA(cudaMemcpy(dw.ptr, weights, (size_t)m * 3 * sizeof(double), cudaMemcpyHostToDevice));
  }
  stencil_finalize(s.get(), di.as<int32_t>(), dw.as<double>(), 0);
  *out_stencil = registry_put(s.release());
  SG_API_END
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

int32_t sg_remap_apply(uint64_t stencil, const uint64_t* src_fields, const uint64_t* dst_fields,
                       int32_t nfields, int32_t variant, uint64_t stream) {
  SG_API_BEGIN
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  SG_REQUIRE(nfields >= 1, "nfields must be >= 1");
  SG_REQUIRE(src_fields && dst_fields, "null field arrays");
  DeviceScope ds(s->device);
  cudaStream_t st = as_stream(stream);
  int32_t levels = -1;
  std::vector<Field*> src(nfields), dst(nfields);
  bool even_pitch = true;
  for (int f = 0; f < nfields; ++f) {
    src[f] = get<Field>(src_fields[f], ObjKind::Field);
    dst[f] = get<Field>(dst_fields[f], ObjKind::Field);
    // exact reference messages, interp.py:208-217
    if (src[f]->npts != s->source_nnodes)
      throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: source field has %lld points, weights expect %lld",
                  (long long)src[f]->npts, (long long)s->source_nnodes);
    if (dst[f]->npts != s->m)
      throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: target field has %lld points, weights cover %lld",
                  (long long)dst[f]->npts, (long long)s->m);
    if (src[f]->levels != dst[f]->levels) throw_error(SG_DOMAIN_ERROR, "ShapeMismatch: level counts differ");
    SG_REQUIRE(src[f]->itemsize == 8 && dst[f]->itemsize == 8, "apply_remap on device needs real64 fields");
    SG_REQUIRE(src[f]->device == s->device && dst[f]->device == s->device,
               "fields and stencil live on different devices");
    if (levels < 0) levels = src[f]->levels;
    SG_REQUIRE(src[f]->levels == levels, "all field pairs of one call must have equal levels");
    even_pitch = even_pitch && (src[f]->pitch % 2 == 0) && (dst[f]->pitch % 2 == 0);
  }
  if (s->m == 0) return SG_OK;
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  for (int f0 = 0; f0 < nfields; f0 += kMaxFields) {
    ApplyArgs a{};
    a.idx = s->idx.as<int4>();
    a.w = s->w.as<double4>();
    a.m = s->m;
    a.levels = levels;
    a.nfields = std::min(kMaxFields, nfields - f0);
    for (int f = 0; f < a.nfields; ++f) {
      a.src[f] = src[f0 + f]->buf.as<double>();
      a.dst[f] = dst[f0 + f]->buf.as<double>();
      a.src_pitch[f] = src[f0 + f]->pitch;
      a.dst_pitch[f] = dst[f0 + f]->pitch;
    }
    const int nvec = (levels + 1) / 2;
    const uint32_t row_bytes = (uint32_t)(((int64_t)levels * 8 + 15) / 16 * 16);
    bool bulk_ok = even_pitch && levels >= 2 && variant == 2;
    for (int f = 0; f < a.nfields && bulk_ok; ++f) bulk_ok = a.src_pitch[f] * 8 >= (int64_t)row_bytes;
    if (bulk_ok) {
      const int row_elems = (int)(row_bytes / 8);
      const size_t smem = (size_t)kStages * 3 * kTile * row_elems * sizeof(double);
      SG_REQUIRE(smem <= 200 * 1024, "levels too large for the bulk-copy variant");
      SG_CUDA(cudaFuncSetAttribute(apply_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, apply_bulk, kV2Threads, smem));
      per_sm = std::max(per_sm, 1);
      const int64_t nwork = (s->m + kTile - 1) / kTile * a.nfields;
      const int64_t grid = std::min<int64_t>((int64_t)g_num_sms * per_sm, nwork);
      apply_bulk<<<(unsigned)grid, kV2Threads, smem, st>>>(a, row_elems, row_bytes);
    } else if (levels <= 8) {
      apply_thread_short<<<(unsigned)((s->m + 255) / 256), 256, 0, st>>>(a);
    } else if (!even_pitch) {
      apply_warp_scalar<<<(unsigned)((s->m + 7) / 8), 256, 0, st>>>(a);
    } else {
      const unsigned grid = (unsigned)((s->m + 7) / 8);  // 8 warps per block
      const int iters = (nvec + 31) / 32;
      switch (iters) {
        case 1: apply_warp_v2<1><<<grid, 256, 0, st>>>(a); break;
        case 2: apply_warp_v2<2><<<grid, 256, 0, st>>>(a); break;
        case 3: apply_warp_v2<3><<<grid, 256, 0, st>>>(a); break;
        case 4: apply_warp_v2<4><<<grid, 256, 0, st>>>(a); break;
        default: apply_warp_scalar<<<grid, 256, 0, st>>>(a); break;
      }
    }
    SG_CUDA_LAUNCH();
  }
  SG_API_END
}

}  // extern "C"
