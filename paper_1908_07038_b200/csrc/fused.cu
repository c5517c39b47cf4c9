// Fused halo exchange + apply over peer memory.
//
// In the reference the remap of a partition needs its ghost rows, so the pipeline is
// halo_exchange (functionspace.py:107-118) then apply_remap (interp.py:206-228).  The ghost
// rows are only read by the stencils of the boundary targets, so on B200 the two steps fuse:
// this kernel applies targets [t0, t1) and, for every stencil node that is a ghost, reads the
// row straight from its owner's field through a peer pointer (same device, NVLink P2P in one
// process, or a CUDA-IPC mapping) — no pack, no transfer buffer, no unpack, no ghost write.
// Local rows [0, plan.ghost_lo) are read from the local field; a ghost row r maps to
// (plan.ghost_slot[r - ghost_lo], plan.ghost_row[r - ghost_lo]) = (owner slot, owner row).
// Arithmetic identical to the apply kernels (bitwise equal to interp.py:219-223).
#include <vector>

#include "plan.cuh"
#include "stencil.cuh"

namespace sg {
namespace {

struct PeerRows {
  const double* base[kMaxPeers];
  int64_t pitch[kMaxPeers];
};

struct FusedArgs {
  const int4* idx;
  const double2* w;  // double4 as two double2
  int64_t t0, t1;
  const int32_t* list;  // optional: target = list[position]
  int k;
  int levels;
  const double* src;
  int64_t src_pitch;
  double* dst;
  int64_t dst_pitch;
  int64_t ghost_lo;
  const int32_t* ghost_slot;
  const int32_t* ghost_row;
  PeerRows peers;
};

__device__ __forceinline__ const double* row_ptr(const FusedArgs& a, int n) {
  if (n < a.ghost_lo) return a.src + (int64_t)n * a.src_pitch;
  const int g = n - (int)a.ghost_lo;
  const int s = __ldg(a.ghost_slot + g);
  return a.peers.base[s] + (int64_t)__ldg(a.ghost_row + g) * a.peers.pitch[s];
}

__device__ __forceinline__ double combine(double w0, double w1, double w2, double x, double y, double z) {
  return __dadd_rn(__dadd_rn(__dmul_rn(w0, x), __dmul_rn(w1, y)), __dmul_rn(w2, z));
}

template <int ITERS>
__global__ void __launch_bounds__(256) apply_fused(FusedArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t pos = a.t0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (pos >= a.t1) return;
  const int64_t t = a.list ? (int64_t)__ldg(a.list + pos) : pos;
  const int4 id = __ldg(a.idx + t);
  const double2 wa = __ldg(a.w + 2 * t), wb = __ldg(a.w + 2 * t + 1);
  const double* r0 = row_ptr(a, id.x);
  const double* r1 = row_ptr(a, id.y);
  const double* r2 = row_ptr(a, id.z);
  const double* r3 = a.k == 4 ? row_ptr(a, id.w) : r0;
  double* out = a.dst + t * a.dst_pitch;
  double v0[ITERS], v1[ITERS], v2[ITERS], v3[ITERS];
#pragma unroll
  for (int i = 0; i < ITERS; ++i) {
    const int l = lane + 32 * i;
    if (l < a.levels) {
      v0[i] = r0[l];
      v1[i] = r1[l];
      v2[i] = r2[l];
      v3[i] = a.k == 4 ? r3[l] : 0.0;
    }
  }
#pragma unroll
  for (int i = 0; i < ITERS; ++i) {
    const int l = lane + 32 * i;
    if (l < a.levels) {
      double o = combine(wa.x, wa.y, wb.x, v0[i], v1[i], v2[i]);
      if (a.k == 4) o = __dadd_rn(o, __dmul_rn(wb.y, v3[i]));
      __stcs(out + l, o);
    }
  }
}

__global__ void __launch_bounds__(256) apply_fused_loop(FusedArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t pos = a.t0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (pos >= a.t1) return;
  const int64_t t = a.list ? (int64_t)__ldg(a.list + pos) : pos;
  const int4 id = __ldg(a.idx + t);
  const double2 wa = __ldg(a.w + 2 * t), wb = __ldg(a.w + 2 * t + 1);
  const double *r0 = row_ptr(a, id.x), *r1 = row_ptr(a, id.y), *r2 = row_ptr(a, id.z);
  const double* r3 = a.k == 4 ? row_ptr(a, id.w) : r0;
  double* out = a.dst + t * a.dst_pitch;
  for (int l = lane; l < a.levels; l += 32) {
    double o = combine(wa.x, wa.y, wb.x, r0[l], r1[l], r2[l]);
    if (a.k == 4) o = __dadd_rn(o, __dmul_rn(wb.y, r3[l]));
    __stcs(out + l, o);
  }
}

}  // namespace
}  // namespace sg

using namespace sg;

namespace {

void fused_impl(uint64_t stencil, uint64_t plan, uint64_t src_field, uint64_t dst_field, int64_t t0, int64_t t1,
                const int32_t* list, const uint64_t* peer_ptrs, const int64_t* peer_pitch_elems, uint64_t stream) {
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  Plan* p = get<Plan>(plan, ObjKind::Plan);
  Field* src = get<Field>(src_field, ObjKind::Field);
  Field* dst = get<Field>(dst_field, ObjKind::Field);
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
  SG_REQUIRE(src->device == s->device && dst->device == s->device && p->device == s->device,
             "stencil, plan and fields live on different devices");
  const size_t np = p->peers.size();
  SG_REQUIRE(np == 0 || (peer_ptrs && peer_pitch_elems), "null peer arrays");
  SG_REQUIRE(p->recv_off.back() == 0 || p->has_remote,
             "plan has ghosts without an owner row (recv_remote); the fused apply needs them");
  FusedArgs a{};
  a.idx = s->idx.as<int4>();
  a.w = s->w.as<double2>();
  a.t0 = t0;
  a.t1 = t1;
  a.list = list;
  a.k = s->k;
  a.levels = src->levels;
  a.src = src->buf.as<double>();
  a.src_pitch = src->pitch;
  a.dst = dst->buf.as<double>();
  a.dst_pitch = dst->pitch;
  a.ghost_lo = p->ghost_lo;
  a.ghost_slot = p->ghost_slot.as<int32_t>();
  a.ghost_row = p->ghost_row.as<int32_t>();
  for (size_t i = 0; i < np; ++i) {
    a.peers.base[i] = reinterpret_cast<const double*>(peer_ptrs[i]);
    a.peers.pitch[i] = peer_pitch_elems[i];
  }
  const int64_t m = t1 - t0;
  if (m <= 0) return;
  DeviceScope ds(s->device);
  const unsigned grid = (unsigned)((m + 1) / 2);  // 2 warps (targets) per block, like apply.cu
  cudaStream_t st = as_stream(stream);
  switch ((a.levels + 31) / 32) {
    case 1: apply_fused<1><<<grid, 64, 0, st>>>(a); break;
    case 2: apply_fused<2><<<grid, 64, 0, st>>>(a); break;
    case 3: apply_fused<3><<<grid, 64, 0, st>>>(a); break;
    case 4: apply_fused<4><<<grid, 64, 0, st>>>(a); break;
    case 5: apply_fused<5><<<grid, 64, 0, st>>>(a); break;
    default: apply_fused_loop<<<grid, 64, 0, st>>>(a); break;
  }
  SG_CUDA_LAUNCH();
}

}  // namespace

extern "C" {

int32_t sg_remap_apply_fused(uint64_t stencil, uint64_t plan, uint64_t src_field, uint64_t dst_field, int64_t t0,
                             int64_t t1, const uint64_t* peer_ptrs, const int64_t* peer_pitch_elems, uint64_t stream) {
  SG_API_BEGIN
  Stencil* s = get<Stencil>(stencil, ObjKind::Stencil);
  SG_REQUIRE(0 <= t0 && t0 <= t1 && t1 <= s->m, "target range outside [0, %lld)", (long long)s->m);
  fused_impl(stencil, plan, src_field, dst_field, t0, t1, nullptr, peer_ptrs, peer_pitch_elems, stream);
  SG_API_END
}

int32_t sg_remap_apply_fused_list(uint64_t stencil, uint64_t plan, uint64_t src_field, uint64_t dst_field,
                                  const int32_t* dev_targets, int64_t count, const uint64_t* peer_ptrs,
                                  const int64_t* peer_pitch_elems, uint64_t stream) {
  SG_API_BEGIN
  SG_REQUIRE(count >= 0 && (count == 0 || dev_targets), "bad target list");
  fused_impl(stencil, plan, src_field, dst_field, 0, count, dev_targets, peer_ptrs, peer_pitch_elems, stream);
  SG_API_END
}

}  // extern "C"
