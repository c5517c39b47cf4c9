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


// 16-B loads where the row is 16-B aligned (even rows at L odd), warp per run piece
__global__ void g_runs16(const double* __restrict__ host, const int2* __restrict__ runs, const int64_t* __restrict__ dst0,
                         double* __restrict__ out, int nruns, int L) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nruns; r += (gridDim.x * blockDim.x) >> 5) {
    const int2 run = runs[r];
    const double* s = host + (int64_t)run.x * L;
    double* d = out + dst0[r] * L;
    int64_t n = (int64_t)run.y * L;
    int head = (reinterpret_cast<uintptr_t>(s) & 15) ? 1 : 0;
    if (head && lane == 0) d[0] = s[0];
    s += head; d += head; n -= head;
    const int64_t n2 = n / 2;
    const double2* s2 = reinterpret_cast<const double2*>(s);
    for (int64_t i = lane; i < n2; i += 32 * 4) {
      double2 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = (i + 32 * k < n2) ? s2[i + 32 * k] : make_double2(0, 0);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i + 32 * k < n2) { d[2 * (i + 32 * k)] = v[k].x; d[2 * (i + 32 * k) + 1] = v[k].y; }
    }
    if ((n & 1) && lane == 0) d[n - 1] = s[n - 1];
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* d, const void* s, uint32_t b, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(d)), "l"(s), "r"(b), "r"(smem_u32(bar)) : "memory");
}

// TMA: producer thread bulk-copies the 16-B aligned superset of a run piece (<= PIECE rows)
// host -> smem; 4 consumer warps copy smem -> compact rows.  STAGES-deep ring.
constexpr int PIECE = 12, STAGES = 4;
__global__ void __launch_bounds__(160) g_tma(const double* __restrict__ host, const int2* __restrict__ pieces,
                                             const int64_t* __restrict__ pdst, double* __restrict__ out, int npieces,
                                             int L, int slot) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + STAGES;
  double* ring = reinterpret_cast<double*>(sm + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 4) {
    if (lane != 0) return;
    int it = 0;
    for (int p = blockIdx.x; p < npieces; p += gridDim.x, ++it) {
      const int st = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[st], ((it / STAGES) - 1) & 1);
      const int2 pc = pieces[p];
      const uintptr_t a = reinterpret_cast<uintptr_t>(host + (int64_t)pc.x * L);
      const uintptr_t s0 = a & ~uintptr_t(15), s1 = (a + (uintptr_t)pc.y * L * 8 + 15) & ~uintptr_t(15);
      mbar_expect_tx(&full[st], (uint32_t)(s1 - s0));
      bulk_g2s(ring + (size_t)st * slot, reinterpret_cast<const void*>(s0), (uint32_t)(s1 - s0), &full[st]);
    }
    return;
  }
  int it = 0;
  for (int p = blockIdx.x; p < npieces; p += gridDim.x, ++it) {
    const int st = it % STAGES;
    mbar_wait(&full[st], (it / STAGES) & 1);
    const int2 pc = pieces[p];
    const int off = (int)((reinterpret_cast<uintptr_t>(host + (int64_t)pc.x * L) & 15) >> 3);
    const double* b = ring + (size_t)st * slot + off;
    double* d = out + pdst[p] * L;
    const int n = pc.y * L;
    for (int i = threadIdx.x; i < n; i += 128) d[i] = b[i];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
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
  std::vector<int2> pieces;
  std::vector<int64_t> pdst;
  for (size_t i = 0; i < runs.size(); ++i)
    for (int q = 0; q < runs[i].y; q += PIECE) {
      pieces.push_back(make_int2(runs[i].x + q, std::min(PIECE, runs[i].y - q)));
      pdst.push_back(dst0[i] + q);
    }
  int2* dpieces; int64_t* dpdst;
  CK(cudaMalloc(&dpieces, pieces.size() * 8)); CK(cudaMemcpy(dpieces, pieces.data(), pieces.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dpdst, pdst.size() * 8)); CK(cudaMemcpy(dpdst, pdst.data(), pdst.size() * 8, cudaMemcpyHostToDevice));
  const int slot = PIECE * L + 4;
  const size_t smem = 128 + (size_t)STAGES * slot * 8;
  CK(cudaFuncSetAttribute(g_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const double gb = (double)U * L * 8;
  printf("{\"U\": %lld, \"runs\": %zu, \"gather_GB\": %.3f}\n", (long long)U, runs.size(), gb / 1e9);
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, c;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&c));
  for (int variant = 1; variant < 5; ++variant)
    for (int gm : {1, 2, 4, 8}) {
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
          else if (variant == 2) g_runs<<<grid, 256, 0, s1>>>(hd, druns, ddst0, out, (int)runs.size(), L);
          else if (variant == 3) g_runs16<<<grid, 256, 0, s1>>>(hd, druns, ddst0, out, (int)runs.size(), L);
          else g_tma<<<grid, 160, smem, s1>>>(hd, dpieces, dpdst, out, (int)pieces.size(), L, slot);
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
