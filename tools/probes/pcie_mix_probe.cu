// PCIe probe: does a kernel reading pinned host memory (zero-copy, 1096-B rows, 77 % of the
// rows as at cfg3) add link throughput on top of a concurrent DMA h2d, or only share it?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pcie_mix_probe pcie_mix_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void zc_read(const double* __restrict__ host, double* __restrict__ dev, int64_t rows, int levels) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if ((r * 2654435761u) % 100 < 23) continue;  // skip ~23 % of the rows
    const double* src = host + r * levels;
    double* dst = dev + r * levels;
    for (int l = lane; l < levels; l += 32) dst[l] = src[l];
  }
}

int main() {
  const int L = 137;
  const size_t bytes = (size_t)2 << 30;
  const int64_t rows = bytes / (L * 8);
  double *ha, *hb, *da, *db, *hbd;
  CK(cudaHostAlloc(&ha, bytes, cudaHostAllocPortable));
  CK(cudaHostAlloc(&hb, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostGetDevicePointer(&hbd, hb, 0));
  CK(cudaMalloc(&da, bytes));
  CK(cudaMalloc(&db, bytes));
  for (size_t i = 0; i < bytes / 8; i += 512) { ha[i] = 1.0; hb[i] = 2.0; }
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  int sms = 148;
  const double zc_bytes = (double)rows * 0.77 * L * 8;
  for (int grid_mult : {2, 4, 8, 16}) {
    for (int pass = 0; pass < 2; ++pass) {
      float t_dma, t_zc, t_both;
      CK(cudaEventRecord(a, s1)); CK(cudaMemcpyAsync(da, ha, bytes, cudaMemcpyHostToDevice, s1));
      CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&t_dma, a, b));
      CK(cudaEventRecord(a, s2)); zc_read<<<sms * grid_mult, 256, 0, s2>>>(hbd, db, rows, L);
      CK(cudaEventRecord(b, s2)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&t_zc, a, b));
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, 0));
      cudaEvent_t fork; CK(cudaEventCreate(&fork)); CK(cudaEventRecord(fork, 0));
      CK(cudaStreamWaitEvent(s1, fork, 0)); CK(cudaStreamWaitEvent(s2, fork, 0));
      CK(cudaMemcpyAsync(da, ha, bytes, cudaMemcpyHostToDevice, s1));
      zc_read<<<sms * grid_mult, 256, 0, s2>>>(hbd, db, rows, L);
      cudaEvent_t j1, j2; CK(cudaEventCreate(&j1)); CK(cudaEventCreate(&j2));
      CK(cudaEventRecord(j1, s1)); CK(cudaEventRecord(j2, s2));
      CK(cudaStreamWaitEvent(0, j1, 0)); CK(cudaStreamWaitEvent(0, j2, 0));
      CK(cudaEventRecord(b, 0)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&t_both, a, b));
      if (pass)
        printf("{\"grid\": %d, \"dma_GBs\": %.1f, \"zc_GBs\": %.1f, \"both_ms\": %.1f, \"both_GBs\": %.1f, \"serial_ms\": %.1f}\n",
               sms * grid_mult, bytes / t_dma / 1e6, zc_bytes / t_zc / 1e6, t_both, (bytes + zc_bytes) / t_both / 1e6,
               t_dma + t_zc);
    }
  }
  return 0;
}
