// PCIe probe for a GPU-side gather of referenced source rows out of pinned, mapped host memory
// into a compact device buffer (the "gather" host-execute mode): read rate of several kernel
// shapes, and whether a concurrent d2h DMA (the target rows going back) slows it.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pcie_gather_probe pcie_gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// warp per compact row, 8-B loads
__global__ void g_warp(const double* __restrict__ host, const int* __restrict__ rows, double* __restrict__ out,
                       int64_t nrows, int L) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < nrows;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double* s = host + (int64_t)rows[u] * L;
    double* d = out + u * L;
    for (int l = lane; l < L; l += 32) d[l] = s[l];
  }
}

// warp per compact row, all loads of the row issued before the stores (ILP 5 at L=137)
template <int IT>
__global__ void g_warp_ilp(const double* __restrict__ host, const int* __restrict__ rows, double* __restrict__ out,
                           int64_t nrows, int L) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < nrows;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double* s = host + (int64_t)rows[u] * L;
    double* d = out + u * L;
    double v[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) v[i] = (lane + 32 * i < L) ? s[lane + 32 * i] : 0.0;
#pragma unroll
    for (int i = 0; i < IT; ++i)
      if (lane + 32 * i < L) d[lane + 32 * i] = v[i];
  }
}

// runs of consecutive referenced rows copied as flat 16-B words where aligned
__global__ void g_runs(const double* __restrict__ host, const int2* __restrict__ runs, const int64_t* __restrict__ dst0,
                       double* __restrict__ out, int nruns, int L) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nruns; r += (gridDim.x * blockDim.x) >> 5) {
    const int2 run = runs[r];  // (first source row, rows)
    const double* s = host + (int64_t)run.x * L;
    double* d = out + dst0[r] * L;
    const int64_t n = (int64_t)run.y * L;
    for (int64_t i = lane; i < n; i += 32 * 4) {
      double v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = (i + 32 * k < n) ? s[i + 32 * k] : 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i + 32 * k < n) d[i + 32 * k] = v[k];
    }
  }
}

int main() {
  const int L = 137;
  const int64_t n = 6599682;  // O1280 + poles
  const size_t bytes = (size_t)n * L * 8;
  double *h, *hd, *out, *dtgt, *htgt;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  const size_t tb = (size_t)1661440 * L * 8;
  CK(cudaHostAlloc(&htgt, tb, cudaHostAllocPortable));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMalloc(&dtgt, tb));
  for (size_t i = 0; i < bytes / 8; i += 512) h[i] = 1.0;
  // referenced rows: isolated single skips, ~23 % (as at O1280->O640)
  std::vector<int> rows;
  std::vector<int2> runs;
  std::vector<int64_t> dst0;
  for (int64_t r = 0; r < n; ++r) {
    if (((uint64_t)r * 2654435761u) % 100 < 23) continue;
    if (!runs.empty() && runs.back().x + runs.back().y == r) runs.back().y++;
    else { runs.push_back(make_int2((int)r, 1)); dst0.push_back((int64_t)rows.size()); }
    rows.push_back((int)r);
  }
  const int64_t U = rows.size();
  int *drows; int2* druns; int64_t* ddst0;
  CK(cudaMalloc(&drows, U * 4)); CK(cudaMemcpy(drows, rows.data(), U * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&druns, runs.size() * 8)); CK(cudaMemcpy(druns, runs.data(), runs.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&ddst0, dst0.size() * 8)); CK(cudaMemcpy(ddst0, dst0.data(), dst0.size() * 8, cudaMemcpyHostToDevice));
  const double gb = (double)U * L * 8;
  printf("{\"U\": %lld, \"runs\": %zu, \"gather_GB\": %.3f}\n", (long long)U, runs.size(), gb / 1e9);
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, c;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&c));
  for (int variant = 0; variant < 3; ++variant)
    for (int gm : {2, 8, 32}) {
      for (int with_d2h = 0; with_d2h < 2; ++with_d2h) {
        float best = 1e30f;
        for (int rep = 0; rep < 2; ++rep) {
          CK(cudaDeviceSynchronize());
          CK(cudaEventRecord(a, s1));
          CK(cudaStreamWaitEvent(s2, a, 0));
          if (with_d2h) CK(cudaMemcpyAsync(htgt, dtgt, tb, cudaMemcpyDeviceToHost, s2));
          const int grid = 148 * gm;
          if (variant == 0) g_warp<<<grid, 256, 0, s1>>>(hd, drows, out, U, L);
          else if (variant == 1) g_warp_ilp<5><<<grid, 256, 0, s1>>>(hd, drows, out, U, L);
          else g_runs<<<grid, 256, 0, s1>>>(hd, druns, ddst0, out, (int)runs.size(), L);
          CK(cudaEventRecord(b, s1));
          CK(cudaEventRecord(c, s2));
          CK(cudaStreamWaitEvent(s1, c, 0));
          CK(cudaEventSynchronize(b));
          float t; CK(cudaEventElapsedTime(&t, a, b));
          if (t < best) best = t;
        }
        CK(cudaGetLastError());
        printf("{\"variant\": %d, \"grid\": %d, \"with_d2h\": %d, \"ms\": %.2f, \"GBs\": %.1f}\n", variant, 148 * gm,
               with_d2h, best, gb / best / 1e6);
      }
    }
  return 0;
}
