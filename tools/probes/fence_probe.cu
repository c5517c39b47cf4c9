// Cost of the memory-model operations the signalled step / exchange use, on one B200:
// a 1-thread kernel doing st.release.sys / st.release.gpu / fence.sc.sys / plain store, and a
// kernel whose N blocks each do one ld.acquire.sys (or .gpu, or volatile) — after a 1 GiB
// write (dirty L2) or after an idle gap.  CUDA events, median of 20.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/fence_probe tools/probes/fence_probe.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k_release_sys(unsigned long long* p) { asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(1ull) : "memory"); }
__global__ void k_release_gpu(unsigned long long* p) { asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(1ull) : "memory"); }
__global__ void k_fence_sc_sys(unsigned long long* p) { __threadfence_system(); *p = 1; }
__global__ void k_plain(unsigned long long* p) { *(volatile unsigned long long*)p = 1; }
__global__ void k_relaxed_sys(unsigned long long* p) { asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(1ull) : "memory"); }
template <int MODE>
__global__ void k_acquire(const unsigned long long* p, unsigned long long* out) {
  if (threadIdx.x) return;
  unsigned long long v;
  if (MODE == 0) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else if (MODE == 1) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else v = *(volatile const unsigned long long*)p;
  if (v == 12345) out[blockIdx.x] = v;
}
__global__ void dirty(float4* a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    a[i] = make_float4(1, 2, 3, 4);
}

template <class F>
float med(F launch, float4* big, size_t nbig, bool pre_dirty) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> t;
  for (int r = 0; r < 21; ++r) {
    if (pre_dirty) dirty<<<148 * 8, 256>>>(big, nbig);
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r) t.push_back(ms * 1000.f);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main() {
  unsigned long long *flag, *out;
  cudaMalloc(&flag, 64);
  cudaMalloc(&out, 8 << 20);
  size_t nbig = (1ull << 30) / 16;
  float4* big;
  cudaMalloc(&big, nbig * 16);
  for (int d = 0; d < 2; ++d) {
    const char* tag = d ? "after 1 GiB write" : "idle";
    printf("{\"case\": \"%s\", \"empty_us\": %.2f, \"plain_store_us\": %.2f, \"relaxed_sys_store_us\": %.2f, "
           "\"release_gpu_us\": %.2f, \"release_sys_us\": %.2f, \"fence_sc_sys_us\": %.2f, "
           "\"acquire_sys_1600_blocks_us\": %.2f, \"acquire_gpu_1600_blocks_us\": %.2f, \"volatile_1600_blocks_us\": %.2f}\n",
           tag, med([&] { k_plain<<<1, 1>>>(out); }, big, nbig, d) * 0 + med([&] {}, big, nbig, d),
           med([&] { k_plain<<<1, 1>>>(flag); }, big, nbig, d),
           med([&] { k_relaxed_sys<<<1, 1>>>(flag); }, big, nbig, d),
           med([&] { k_release_gpu<<<1, 1>>>(flag); }, big, nbig, d),
           med([&] { k_release_sys<<<1, 1>>>(flag); }, big, nbig, d),
           med([&] { k_fence_sc_sys<<<1, 1>>>(flag); }, big, nbig, d),
           med([&] { k_acquire<0><<<1600, 256>>>(flag, out); }, big, nbig, d),
           med([&] { k_acquire<1><<<1600, 256>>>(flag, out); }, big, nbig, d),
           med([&] { k_acquire<2><<<1600, 256>>>(flag, out); }, big, nbig, d));
  }
  return 0;
}
