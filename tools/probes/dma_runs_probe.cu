// Probe: can the copy engine move the long referenced runs of the cfg3 e2e gather (25 k runs
// of >= 64 rows, ~114 rows x 1096 B each) fast enough, and what does issuing one
// cudaMemcpyAsync per run cost on the host?  Prints one JSON line per setting.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o dma_runs_probe dma_runs_probe.cu -lpthread
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

int main() {
  const size_t row = 1096;
  const int nruns_max = 25000;
  const size_t run_rows = 114, gap_rows = 150;  // runs separated like the cfg3 pattern
  const size_t host_rows = nruns_max * (run_rows + gap_rows);
  char* host = nullptr;
  CK(cudaHostAlloc(&host, host_rows * row, cudaHostAllocMapped));
  for (size_t i = 0; i < host_rows * row; i += 4096) host[i] = (char)i;
  char* dev = nullptr;
  CK(cudaMalloc(&dev, (size_t)nruns_max * run_rows * row));
  for (int nthreads : {1}) {
    for (int nruns : {5000, 25000}) {
      std::vector<cudaStream_t> st(nthreads);
      for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaDeviceSynchronize());
        auto t0 = std::chrono::steady_clock::now();
        std::vector<double> issue(nthreads);
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t)
          th.emplace_back([&, t] {
            auto a = std::chrono::steady_clock::now();
            for (int r = t; r < nruns; r += nthreads)
              cudaMemcpyAsync(dev + (size_t)r * run_rows * row, host + (size_t)r * (run_rows + gap_rows) * row,
                              run_rows * row, cudaMemcpyHostToDevice, st[t]);
            issue[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
          });
        for (auto& x : th) x.join();
        CK(cudaDeviceSynchronize());
        double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        double bytes = (double)nruns * run_rows * row;
        double imax = 0;
        for (double v : issue) imax = imax > v ? imax : v;
        if (rep == 2)
          printf("{\"threads\": %d, \"runs\": %d, \"issue_ms\": %.2f, \"us_per_call\": %.3f, \"total_ms\": %.2f, \"GBs\": %.2f}\n",
                 nthreads, nruns, imax * 1e3, imax * 1e6 / (nruns / nthreads), total * 1e3, bytes / total / 1e9);
      }
      for (auto& s : st) CK(cudaStreamDestroy(s));
    }
  }
  // the same copies captured once into a CUDA graph (one or two chains), replayed
  for (int chains : {1, 2, 4}) {
    for (int nruns : {5000, 25000}) {
      std::vector<cudaStream_t> st(chains);
      for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      cudaEvent_t fork, join[4];
      CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      for (int c = 0; c < chains; ++c) CK(cudaEventCreateWithFlags(&join[c], cudaEventDisableTiming));
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st[0], cudaStreamCaptureModeGlobal));
      CK(cudaEventRecord(fork, st[0]));
      for (int c = 1; c < chains; ++c) CK(cudaStreamWaitEvent(st[c], fork, 0));
      for (int r = 0; r < nruns; ++r)
        CK(cudaMemcpyAsync(dev + (size_t)r * run_rows * row, host + (size_t)r * (run_rows + gap_rows) * row,
                           run_rows * row, cudaMemcpyHostToDevice, st[r % chains]));
      for (int c = 1; c < chains; ++c) {
        CK(cudaEventRecord(join[c], st[c]));
        CK(cudaStreamWaitEvent(st[0], join[c], 0));
      }
      CK(cudaStreamEndCapture(st[0], &g));
      cudaGraphExec_t ge;
      auto ti = std::chrono::steady_clock::now();
      CK(cudaGraphInstantiate(&ge, g, 0));
      double inst = std::chrono::duration<double>(std::chrono::steady_clock::now() - ti).count();
      for (int rep = 0; rep < 4; ++rep) {
        CK(cudaDeviceSynchronize());
        auto t0 = std::chrono::steady_clock::now();
        CK(cudaGraphLaunch(ge, st[0]));
        double launch = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        CK(cudaStreamSynchronize(st[0]));
        double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (rep == 3)
          printf("{\"graph_chains\": %d, \"runs\": %d, \"instantiate_ms\": %.1f, \"launch_ms\": %.3f, \"total_ms\": %.2f, \"GBs\": %.2f}\n",
                 chains, nruns, inst * 1e3, launch * 1e3, total * 1e3, (double)nruns * run_rows * row / total / 1e9);
      }
      CK(cudaGraphExecDestroy(ge));
      CK(cudaGraphDestroy(g));
      for (auto& s : st) CK(cudaStreamDestroy(s));
    }
  }
  // reference: one big copy of the same bytes
  CK(cudaDeviceSynchronize());
  auto t0 = std::chrono::steady_clock::now();
  CK(cudaMemcpyAsync(dev, host, (size_t)nruns_max * run_rows * row, cudaMemcpyHostToDevice, 0));
  CK(cudaDeviceSynchronize());
  double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("{\"one_copy_GBs\": %.2f}\n", (double)nruns_max * run_rows * row / total / 1e9);
  return 0;
}
