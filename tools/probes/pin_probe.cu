// Cost of page-locked host mirrors of cfg3 size (7.23 GB): cudaHostAlloc (+ device memset),
// versus mmap + transparent huge pages + parallel first touch + cudaHostRegister.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o pin_probe pin_probe.cu -lpthread
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t bytes = 6599682ull * 137 * 8;
  cudaFree(0);
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now();
    void* p = nullptr;
    cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
    double t1 = now();
    void* dp = nullptr;
    cudaHostGetDevicePointer(&dp, p, 0);
    cudaMemset(dp, 0, bytes);
    cudaDeviceSynchronize();
    double t2 = now();
    cudaFreeHost(p);
    double t3 = now();
    printf("{\"path\": \"cudaHostAlloc\", \"alloc_s\": %.3f, \"memset_s\": %.3f, \"free_s\": %.3f}\n", t1 - t0, t2 - t1, t3 - t2);

    for (int nth : {1, 8, 16}) {
      for (int thp : {0, 1}) {
        t0 = now();
        void* q = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (thp) madvise(q, bytes, MADV_HUGEPAGE);
        std::vector<std::thread> th;
        for (int i = 0; i < nth; ++i)
          th.emplace_back([&, i] {
            const size_t a = bytes * i / nth, b = bytes * (i + 1) / nth;
            for (size_t o = a; o < b; o += 4096) static_cast<volatile char*>(q)[o] = 0;
          });
        for (auto& x : th) x.join();
        t1 = now();
        cudaError_t e = cudaHostRegister(q, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
        t2 = now();
        cudaHostUnregister(q);
        munmap(q, bytes);
        t3 = now();
        printf("{\"path\": \"mmap+touch+register\", \"threads\": %d, \"thp\": %d, \"touch_s\": %.3f, \"register_s\": %.3f, "
               "\"ok\": %d, \"free_s\": %.3f}\n", nth, thp, t1 - t0, t2 - t1, e == cudaSuccess, t3 - t2);
      }
    }
  }
  return 0;
}
