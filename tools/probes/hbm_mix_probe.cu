// HBM ceiling for the apply's traffic mix: the same bytes as one cfg3 apply launch
// (O1280 -> O640, 137 levels: 4.98 M source rows read, 1.66 M target rows written, 1096-B dense
// rows), moved by kernels with the same warp-per-target shape as apply_warp_v1 but perfectly
// sequential addresses — so the only difference from the real kernel is the gather pattern.
//   seq3to1 : target t reads rows 3t, 3t+1, 3t+2 of a packed source, writes row t (same
//             arithmetic as the apply).  The apply kernel's ceiling for this read/write mix.
//   read    : the same reads, no writes (one double per warp written to keep them alive).
//   copy    : 1 row read, 1 row written per warp (what MEASURED_PEAKS' copy figure measures).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hbm_mix_probe hbm_mix_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                      \
      return 1;                                                           \
    }                                                                     \
  } while (0)

constexpr int L = 137;
constexpr int IT = 5;

__device__ __forceinline__ double ld(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(256) seq3to1(const double* __restrict__ src, double* __restrict__ dst, int64_t m,
                                               double w0, double w1, double w2) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= m) return;
  const double* r0 = src + (3 * t) * L;
  const double* r1 = r0 + L;
  const double* r2 = r1 + L;
  double v0[IT], v1[IT], v2[IT];
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const int k = lane + 32 * i;
    if (k < L) {
      v0[i] = ld(r0 + k);
      v1[i] = ld(r1 + k);
      v2[i] = ld(r2 + k);
    }
  }
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const int k = lane + 32 * i;
    if (k < L) __stcs(dst + t * L + k, __dadd_rn(__dadd_rn(__dmul_rn(w0, v0[i]), __dmul_rn(w1, v1[i])), __dmul_rn(w2, v2[i])));
  }
}


// variants of seq3to1's shape (same bytes)
// ST: 0 st.global.cs, 1 plain st, 2 st.global.L1::no_allocate ; ORD: 0 interleaved, 1 row by row
template <int ST, int ORD>
__global__ void __launch_bounds__(256) seqv(const double* __restrict__ src, double* __restrict__ dst, int64_t m,
                                            double w0, double w1, double w2) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= m) return;
  const double* r0 = src + (3 * t) * L;
  double v[3][IT];
  if (ORD == 1) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int i = 0; i < IT; ++i)
        if (lane + 32 * i < L) v[r][i] = ld(r0 + r * L + lane + 32 * i);
  } else {
#pragma unroll
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int r = 0; r < 3; ++r)
        if (lane + 32 * i < L) v[r][i] = ld(r0 + r * L + lane + 32 * i);
  }
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const int k = lane + 32 * i;
    if (k < L) {
      const double o = __dadd_rn(__dadd_rn(__dmul_rn(w0, v[0][i]), __dmul_rn(w1, v[1][i])), __dmul_rn(w2, v[2][i]));
      double* q = dst + t * L + k;
      if (ST == 0) __stcs(q, o);
      else if (ST == 1) *q = o;
      else asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" :: "l"(q), "d"(o) : "memory");
    }
  }
}

// persistent warps: grid-stride over targets
__global__ void __launch_bounds__(256) seq_persist(const double* __restrict__ src, double* __restrict__ dst, int64_t m,
                                                   double w0, double w1, double w2) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < m; t += nw) {
    const double* r0 = src + (3 * t) * L;
    double v0[IT], v1[IT], v2[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int k = lane + 32 * i;
      if (k < L) {
        v0[i] = ld(r0 + k);
        v1[i] = ld(r0 + L + k);
        v2[i] = ld(r0 + 2 * L + k);
      }
    }
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int k = lane + 32 * i;
      if (k < L) __stcs(dst + t * L + k, __dadd_rn(__dadd_rn(__dmul_rn(w0, v0[i]), __dmul_rn(w1, v1[i])), __dmul_rn(w2, v2[i])));
    }
  }
}

// flat 3-input triad, 16-B vectors, grid-stride: the best case for a 3:1 read:write mix
__global__ void __launch_bounds__(256) triad3(const double2* __restrict__ a, const double2* __restrict__ b,
                                              const double2* __restrict__ c, double2* __restrict__ d, int64_t n,
                                              double w0, double w1, double w2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    double2 x[4], y[4], z[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * stride < n) {
        x[u] = __ldcs(a + i + u * stride);
        y[u] = __ldcs(b + i + u * stride);
        z[u] = __ldcs(c + i + u * stride);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * stride < n) {
        double2 o;
        o.x = __dadd_rn(__dadd_rn(__dmul_rn(w0, x[u].x), __dmul_rn(w1, y[u].x)), __dmul_rn(w2, z[u].x));
        o.y = __dadd_rn(__dadd_rn(__dmul_rn(w0, x[u].y), __dmul_rn(w1, y[u].y)), __dmul_rn(w2, z[u].y));
        __stcs(d + i + u * stride, o);
      }
  }
}

__global__ void __launch_bounds__(256) read3(const double* __restrict__ src, double* __restrict__ dst, int64_t m) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= m) return;
  const double* r0 = src + (3 * t) * L;
  double s = 0;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const int k = lane + 32 * i;
    if (k < L) s += ld(r0 + k) + ld(r0 + L + k) + ld(r0 + 2 * L + k);
  }
  if (s == 12345.678) dst[t] = s;  // never true: keeps the loads
}

__global__ void __launch_bounds__(256) copy1(const double* __restrict__ src, double* __restrict__ dst, int64_t m) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= m) return;
  double v[IT];
#pragma unroll
  for (int i = 0; i < IT; ++i)
    if (lane + 32 * i < L) v[i] = ld(src + t * L + lane + 32 * i);
#pragma unroll
  for (int i = 0; i < IT; ++i)
    if (lane + 32 * i < L) __stcs(dst + t * L + lane + 32 * i, v[i]);
}

int main() {
  const int64_t m = 1661440, U = 3 * m;  // cfg3 targets; 4,984,320 source rows (U = 4,983,053)
  double *src, *dst;
  CK(cudaMalloc(&src, U * L * 8));
  CK(cudaMalloc(&dst, U * L * 8));  // large enough for the copy test's writes
  CK(cudaMemset(src, 0, U * L * 8));
  CK(cudaMemset(dst, 0, U * L * 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 20;
  const unsigned gm = (unsigned)((m + 7) / 8);
  const double mix = (double)(U + m) * L * 8;
  const int64_t n2 = m * L / 2;  // double2 per triad stream
  struct K {
    const char* name;
    double bytes;
  };
  const K ks[] = {{"seq3to1 (apply shape, sequential rows, st.cs)", mix},
                  {"seq3to1 plain stores", mix},
                  {"seq3to1 st.L1::no_allocate", mix},
                  {"seq3to1 row-by-row load order", mix},
                  {"seq3to1 persistent 148x4 blocks", mix},
                  {"seq3to1 persistent 148x8 blocks", mix},
                  {"triad3 flat 16-B streams 148x8 blocks", mix},
                  {"triad3 flat 16-B streams 148x32 blocks", mix},
                  {"read only (apply shape)", (double)U * L * 8},
                  {"copy 1:1 (apply shape)", 2.0 * U * L * 8}};
  for (int kind = 0; kind < 10; ++kind) {
    auto launch = [&] {
      switch (kind) {
        case 0: seq3to1<<<gm, 256>>>(src, dst, m, 0.25, 0.5, 0.25); break;
        case 1: seqv<1, 0><<<gm, 256>>>(src, dst, m, 0.25, 0.5, 0.25); break;
        case 2: seqv<2, 0><<<gm, 256>>>(src, dst, m, 0.25, 0.5, 0.25); break;
        case 3: seqv<0, 1><<<gm, 256>>>(src, dst, m, 0.25, 0.5, 0.25); break;
        case 4: seq_persist<<<148 * 4, 256>>>(src, dst, m, 0.25, 0.5, 0.25); break;
        case 5: seq_persist<<<148 * 8, 256>>>(src, dst, m, 0.25, 0.5, 0.25); break;
        case 6:
        case 7: {
          const double2* a = reinterpret_cast<const double2*>(src);
          triad3<<<148 * (kind == 6 ? 8 : 32), 256>>>(a, a + n2, a + 2 * n2, reinterpret_cast<double2*>(dst), n2, 0.25, 0.5, 0.25);
          break;
        }
        case 8: read3<<<gm, 256>>>(src, dst, m); break;
        default: copy1<<<(unsigned)((U + 7) / 8), 256>>>(src, dst, U); break;
      }
    };
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"bytes\": %.0f, \"GBs\": %.1f}\n", ks[kind].name, ms, ks[kind].bytes,
           ks[kind].bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
