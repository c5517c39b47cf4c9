// Partition-invariant field digest on the device: checksum (functionspace.py:233-254,
// format pkg/README.md:76-94).  For every owned (point, level):
//   key = gid * 0x9E3779B97F4A7C15 + (level + 1) * 0xC2B2AE3D27D4EB4F      (wrapping u64)
//   h   = splitmix64_finalizer(key ^ value_bits)                           (functionspace.py:37-44)
// value_bits = the 8-byte pattern, or the 4-byte pattern zero-extended (functionspace.py:227-230);
// the partial digest is the wrapping u64 sum over the owned rows.  Integer-only: bit-exact.
//
// Indexed row copy for gather_field / scatter_field (functionspace.py:185-224) on the device:
//   dst[dst_idx ? dst_idx[i] : i] = src[src_idx ? src_idx[i] : i],  i in [0, n)
// a warp per row, every lane issuing all its loads before its stores; src / dst may be a
// peer's memory (NVLink P2P in one process, CUDA IPC across processes), so rank 0 assembles
// the global field straight from the ranks' HBM (gather) and every rank pulls its owned rows
// from rank 0's copy of the global array (scatter).
#include <vector>

#include "cuda_util.cuh"

namespace {

constexpr unsigned long long kGamma = 0x9E3779B97F4A7C15ull;
constexpr unsigned long long kLevel = 0xC2B2AE3D27D4EB4Full;
constexpr unsigned long long kM1 = 0xBF58476D1CE4E5B9ull;
constexpr unsigned long long kM2 = 0x94D049BB133111EBull;

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30;
  x *= kM1;
  x ^= x >> 27;
  x *= kM2;
  x ^= x >> 31;
  return x;
}

template <int ITEM>
__global__ void checksum_kernel(const unsigned char* base, int64_t pitch_bytes, int levels, int64_t row0,
                                const int64_t* gids, int64_t nrows, unsigned long long* out) {
  unsigned long long acc = 0;
  const int64_t total = nrows * levels;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / levels;
    const int l = (int)(e - r * levels);
    const unsigned char* p = base + (row0 + r) * pitch_bytes + (int64_t)l * ITEM;
    const unsigned long long bits =
        ITEM == 8 ? *reinterpret_cast<const unsigned long long*>(p) : (unsigned long long)*reinterpret_cast<const unsigned int*>(p);
    const unsigned long long key = (unsigned long long)gids[r] * kGamma + (unsigned long long)(l + 1) * kLevel;
    acc += mix64(key ^ bits);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

template <class W, int UNROLL>
__global__ void __launch_bounds__(256) rows_copy_kernel(char* dst, int64_t dst_pitch, const int64_t* dst_idx,
                                                         const char* src, int64_t src_pitch, const int64_t* src_idx,
                                                         int64_t n, int64_t words) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t di = dst_idx ? __ldg(dst_idx + i) : i, si = src_idx ? __ldg(src_idx + i) : i;
  W* d = reinterpret_cast<W*>(dst + di * dst_pitch);
  const W* s = reinterpret_cast<const W*>(src + si * src_pitch);
  for (int64_t base = 0; base < words; base += 32 * UNROLL) {
    W v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t k = base + lane + 32 * u;
      if (k < words) v[u] = s[k];
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t k = base + lane + 32 * u;
      if (k < words) d[k] = v[u];
    }
  }
}

template <class W>
void launch_rows_copy(char* dst, int64_t dp, const int64_t* di, const char* src, int64_t sp, const int64_t* si,
                      int64_t n, int64_t row_bytes, cudaStream_t st) {
  const int64_t words = row_bytes / (int64_t)sizeof(W);
  const unsigned grid = (unsigned)((n * 32 + 255) / 256);
  rows_copy_kernel<W, 8><<<grid, 256, 0, st>>>(dst, dp, di, src, sp, si, n, words);
}

}  // namespace

using namespace sg;

extern "C" int32_t sg_field_checksum(uint64_t field, int64_t row0, int64_t nrows, const int64_t* gids,
                                     uint64_t* out_partial) {
  SG_API_BEGIN
  Field* f = get<Field>(field, ObjKind::Field);
  SG_REQUIRE(out_partial, "null out pointer");
  SG_REQUIRE(row0 >= 0 && nrows >= 0 && row0 + nrows <= f->npts, "row range outside the field");
  SG_REQUIRE(nrows == 0 || gids, "null gids");
  DeviceScope ds(f->device);
  cudaStream_t st = 0;
  DevBuf dg, dacc;
  dg.alloc(f->device, (size_t)std::max<int64_t>(nrows, 1) * 8);
  dacc.alloc(f->device, 8);
  SG_CUDA(cudaMemsetAsync(dacc.ptr, 0, 8, st));
  if (nrows) {
    SG_CUDA(cudaMemcpyAsync(dg.ptr, gids, (size_t)nrows * 8, cudaMemcpyHostToDevice, st));
    const int64_t total = nrows * f->levels;
    const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
    const int64_t pitch_bytes = f->pitch * f->itemsize;
    if (f->itemsize == 8)
      checksum_kernel<8><<<grid, 256, 0, st>>>(f->buf.as<unsigned char>(), pitch_bytes, f->levels, row0,
                                               dg.as<int64_t>(), nrows, dacc.as<unsigned long long>());
    else
      checksum_kernel<4><<<grid, 256, 0, st>>>(f->buf.as<unsigned char>(), pitch_bytes, f->levels, row0,
                                               dg.as<int64_t>(), nrows, dacc.as<unsigned long long>());
    SG_CUDA_LAUNCH();
  }
  SG_CUDA(cudaMemcpyAsync(out_partial, dacc.ptr, 8, cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  SG_API_END
}

extern "C" int32_t sg_rows_copy(int32_t device, uint64_t dst, int64_t dst_pitch_bytes, const int64_t* dst_idx_dev,
                                uint64_t src, int64_t src_pitch_bytes, const int64_t* src_idx_dev, int64_t n,
                                int64_t row_bytes, uint64_t stream) {
  SG_API_BEGIN
  SG_REQUIRE(n >= 0 && row_bytes >= 0, "negative size");
  if (n == 0 || row_bytes == 0) return SG_OK;
  SG_REQUIRE(dst && src, "null row pointers");
  SG_REQUIRE(row_bytes % 4 == 0 && dst_pitch_bytes >= row_bytes && src_pitch_bytes >= row_bytes,
             "rows must be whole 4-byte words within their pitch");
  DeviceScope ds(device);
  cudaStream_t st = as_stream(stream);
  char* d = reinterpret_cast<char*>(dst);
  const char* s = reinterpret_cast<const char*>(src);
  const uint64_t align = dst | src | (uint64_t)dst_pitch_bytes | (uint64_t)src_pitch_bytes | (uint64_t)row_bytes;
  if (align % 16 == 0)
    launch_rows_copy<int4>(d, dst_pitch_bytes, dst_idx_dev, s, src_pitch_bytes, src_idx_dev, n, row_bytes, st);
  else if (align % 8 == 0)
    launch_rows_copy<unsigned long long>(d, dst_pitch_bytes, dst_idx_dev, s, src_pitch_bytes, src_idx_dev, n,
                                         row_bytes, st);
  else
    launch_rows_copy<unsigned int>(d, dst_pitch_bytes, dst_idx_dev, s, src_pitch_bytes, src_idx_dev, n, row_bytes,
                                   st);
  SG_CUDA_LAUNCH();
  SG_API_END
}
