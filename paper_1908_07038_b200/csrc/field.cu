// Device mirror of a reference Field (field.py:77-162): level-contiguous rows with the
// pitch chosen by field_pitch_elems (dense today).  h2d/d2h move the unpadded host
// (npts, levels) C-order array (field.py:161): one contiguous copy for dense rows, a
// cudaMemcpy2DAsync otherwise.
#include <cstring>
#include <sys/mman.h>

#include <algorithm>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "apply_internal.cuh"
#include "cuda_util.cuh"

using namespace sg;

namespace {
// Large pinned buffers: anonymous mmap backed by transparent huge pages, first-touched by
// several threads, then cudaHostRegister'ed.  ~0.3 s for a 7.2 GB cfg3 mirror against ~3 s for
// cudaHostAlloc, whose 4-KB pages the kernel zero-fills and pins one by one
// (tools/probes/pin_probe.cu, profiles/r01_pin_probe.txt).  Fresh anonymous pages are zero.
constexpr size_t kMmapPinBytes = size_t(64) << 20;
std::mutex g_mm_mu;
std::unordered_map<uintptr_t, size_t> g_mm;  // mmap'ed + registered buffers -> length

void* mmap_pinned(size_t bytes) {
  void* q = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (q == MAP_FAILED) return nullptr;
  madvise(q, bytes, MADV_HUGEPAGE);
  const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int i = 0; i < nth; ++i)
    th.emplace_back([=] {
      const size_t a = bytes * i / nth, b = bytes * (i + 1) / nth;
      for (size_t o = a & ~size_t(4095); o < b; o += 4096)
        if (o >= a) static_cast<volatile char*>(q)[o] = 0;
    });
  for (auto& t : th) t.join();
  if (cudaHostRegister(q, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped) != cudaSuccess) {
    cudaGetLastError();
    munmap(q, bytes);
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_mm_mu);
  g_mm[reinterpret_cast<uintptr_t>(q)] = bytes;
  return q;
}
}  // namespace

extern "C" {

// 16-byte UUID of a device: tells whether two ranks (processes) drive the same physical GPU.
int32_t sg_device_uuid(int32_t device, uint8_t* out_uuid, size_t n) {
  SG_API_BEGIN
  SG_REQUIRE(out_uuid && n >= 16, "buffer must hold 16 bytes");
  cudaDeviceProp prop;
  SG_CUDA(cudaGetDeviceProperties(&prop, device));
  memcpy(out_uuid, prop.uuid.bytes, 16);
  SG_API_END
}

int32_t sg_device_count(int32_t* out_count) {
  SG_API_BEGIN
  SG_REQUIRE(out_count, "null out pointer");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *out_count = n;
  SG_API_END
}

int32_t sg_stream_synchronize(int32_t device, uint64_t stream) {
  SG_API_BEGIN
  DeviceScope ds(device);
  SG_CUDA(cudaStreamSynchronize(as_stream(stream)));
  SG_API_END
}

int32_t sg_field_alloc(int32_t device, int64_t npts, int32_t levels, int32_t itemsize,
                       uint64_t* out_field, int64_t* out_pitch_elems, uint64_t* out_devptr) {
  SG_API_BEGIN
  SG_REQUIRE(out_field, "null out pointer");
  SG_REQUIRE(npts >= 0 && levels >= 1, "bad field shape (%lld, %d)", (long long)npts, levels);
  SG_REQUIRE(itemsize == 4 || itemsize == 8, "itemsize must be 4 or 8");
  DeviceScope ds(device);
  auto f = std::make_unique<Field>();
  f->device = device;
  f->npts = npts;
  f->levels = levels;
  f->itemsize = itemsize;
  f->pitch = field_pitch_elems(levels, itemsize);
  // +16 B slack: the bulk-copy apply reads the 16-B aligned superset of a row, which can
  // reach 8 B past the last dense row
  size_t bytes = (size_t)std::max<int64_t>(npts, 1) * f->pitch * itemsize + 16;
  f->buf.alloc(device, bytes);
  SG_CUDA(cudaMemset(f->buf.ptr, 0, bytes));
  if (out_pitch_elems) *out_pitch_elems = f->pitch;
  if (out_devptr) *out_devptr = reinterpret_cast<uint64_t>(f->buf.ptr);
  *out_field = registry_put(f.release());
  SG_API_END
}

int32_t sg_field_info(uint64_t field, int32_t* out_device, int64_t* out_npts, int32_t* out_levels,
                      int64_t* out_pitch_elems, uint64_t* out_devptr) {
  SG_API_BEGIN
  Field* f = get<Field>(field, ObjKind::Field);
  if (out_device) *out_device = f->device;
  if (out_npts) *out_npts = f->npts;
  if (out_levels) *out_levels = f->levels;
  if (out_pitch_elems) *out_pitch_elems = f->pitch;
  if (out_devptr) *out_devptr = reinterpret_cast<uint64_t>(f->buf.ptr);
  SG_API_END
}

// runs[2r], runs[2r+1] = (row0, nrows): 32-bit words of rows [row0, row0 + nrows) from the
// mapped host array into the same rows of a dense device field; block per run
__global__ void __launch_bounds__(256) copy_runs_kernel(const uint32_t* __restrict__ host, uint32_t* __restrict__ dev,
                                                        const int64_t* __restrict__ runs, int64_t nruns,
                                                        int64_t row_words) {
  for (int64_t r = blockIdx.x; r < nruns; r += gridDim.x) {
    const int64_t w0 = runs[2 * r] * row_words, nw = runs[2 * r + 1] * row_words;
    const uint32_t* s = host + w0;
    uint32_t* d = dev + w0;
    if (((w0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(host) | reinterpret_cast<uintptr_t>(dev)) & 7) == 0) {
      const int64_t n2 = nw >> 1;  // 8-B moves
      for (int64_t i = threadIdx.x; i < n2; i += blockDim.x)
        reinterpret_cast<uint2*>(d)[i] = reinterpret_cast<const uint2*>(s)[i];
      if ((nw & 1) && threadIdx.x == 0) d[nw - 1] = s[nw - 1];
    } else {
      for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) d[i] = s[i];
    }
  }
}

static void copy_rows(Field* f, int64_t row0, int64_t nrows, const void* src_host, void* dst_host,
                      uint64_t stream) {
  SG_REQUIRE(row0 >= 0 && nrows >= 0 && row0 + nrows <= f->npts, "row range [%lld, %lld) outside [0, %lld)",
             (long long)row0, (long long)(row0 + nrows), (long long)f->npts);
  if (nrows == 0) return;
  DeviceScope ds(f->device);
  size_t row_bytes = (size_t)f->levels * f->itemsize;
  size_t pitch_bytes = (size_t)f->pitch * f->itemsize;
  char* dev = f->buf.as<char>() + (size_t)row0 * pitch_bytes;
  if (pitch_bytes == row_bytes) {  // dense rows: one contiguous copy
    const size_t n = row_bytes * (size_t)nrows;
    if (src_host)
      SG_CUDA(cudaMemcpyAsync(dev, src_host, n, cudaMemcpyHostToDevice, as_stream(stream)));
    else
      SG_CUDA(cudaMemcpyAsync(dst_host, dev, n, cudaMemcpyDeviceToHost, as_stream(stream)));
  } else if (src_host) {
    SG_CUDA(cudaMemcpy2DAsync(dev, pitch_bytes, src_host, row_bytes, row_bytes, (size_t)nrows,
                              cudaMemcpyHostToDevice, as_stream(stream)));
  } else {
    SG_CUDA(cudaMemcpy2DAsync(dst_host, row_bytes, dev, pitch_bytes, row_bytes, (size_t)nrows,
                              cudaMemcpyDeviceToHost, as_stream(stream)));
  }
}

int32_t sg_field_h2d(uint64_t field, const void* host, uint64_t stream) {
  SG_API_BEGIN
  Field* f = get<Field>(field, ObjKind::Field);
  SG_REQUIRE(host || f->npts == 0, "null host pointer");
  copy_rows(f, 0, f->npts, host, nullptr, stream);
  SG_API_END
}

int32_t sg_field_d2h(uint64_t field, void* host, uint64_t stream) {
  SG_API_BEGIN
  Field* f = get<Field>(field, ObjKind::Field);
  SG_REQUIRE(host || f->npts == 0, "null host pointer");
  copy_rows(f, 0, f->npts, nullptr, host, stream);
  SG_API_END
}

int32_t sg_field_h2d_rows(uint64_t field, int64_t row0, int64_t nrows, const void* host,
                          uint64_t stream) {
  SG_API_BEGIN
  Field* f = get<Field>(field, ObjKind::Field);
  SG_REQUIRE(host || nrows == 0, "null host pointer");
  copy_rows(f, row0, nrows, host, nullptr, stream);
  SG_API_END
}

// Row runs (row0, nrows) pairs of the full (npts, levels) host array into the same rows of the
// device field: the host-field halo exchange uploads only the rows peers read (the union of
// the send lists: 2-4 runs for bands, ~1,300 for equal regions at O1280 P=8) instead of all
// rows (functionspace.halo_exchange).
int32_t sg_field_h2d_row_runs(uint64_t field, const int64_t* runs, int64_t nruns, const void* host,
                              uint64_t stream) {
  SG_API_BEGIN
  Field* f = get<Field>(field, ObjKind::Field);
  SG_REQUIRE(nruns >= 0 && (runs || nruns == 0), "bad run list");
  SG_REQUIRE(host || nruns == 0, "null host pointer");
  const size_t row_bytes = (size_t)f->levels * f->itemsize;
  for (int64_t r = 0; r < nruns; ++r)
    SG_REQUIRE(runs[2 * r] >= 0 && runs[2 * r + 1] >= 0 && runs[2 * r] + runs[2 * r + 1] <= f->npts,
               "run %lld outside [0, %lld)", (long long)r, (long long)f->npts);
  if (nruns == 0) return SG_OK;
  DeviceScope ds(f->device);
  // many short runs from pinned, mapped host memory (create_field mirrors): one kernel pulls
  // them over PCIe instead of one small DMA per run (equal regions: ~1,300 runs per rank)
  cudaPointerAttributes at{};
  const bool mapped = nruns > 16 && f->pitch == f->levels &&
                      cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost &&
                      at.devicePointer != nullptr;
  cudaGetLastError();
  if (mapped && f->itemsize * f->levels % 8 == 0 && detail::gather_fits((int)(row_bytes / 8))) {
    // rows as doubles: bulk-copy pieces (cp.async.bulk, the e2e gather) into the same rows
    const int words = (int)(row_bytes / 8), prows = detail::gather_piece_rows(words);
    std::vector<int2> pcs;
    std::vector<int64_t> dst;
    for (int64_t r = 0; r < nruns; ++r)
      for (int64_t q = 0; q < runs[2 * r + 1]; q += prows) {
        pcs.push_back(make_int2((int)(runs[2 * r] + q), (int)std::min<int64_t>(prows, runs[2 * r + 1] - q)));
        dst.push_back(runs[2 * r] + q);
      }
    thread_local DevBuf sp, sd;
    if (sp.bytes < pcs.size() * sizeof(int2) || sp.device != f->device)
      sp.alloc(f->device, std::max<size_t>(pcs.size() * sizeof(int2), 4096));
    if (sd.bytes < dst.size() * sizeof(int64_t) || sd.device != f->device)
      sd.alloc(f->device, std::max<size_t>(dst.size() * sizeof(int64_t), 4096));
    cudaStream_t st = as_stream(stream);
    if (!pcs.empty()) {
      SG_CUDA(cudaMemcpyAsync(sp.ptr, pcs.data(), pcs.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
      SG_CUDA(cudaMemcpyAsync(sd.ptr, dst.data(), dst.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      detail::launch_gather_tma(static_cast<const double*>(at.devicePointer), f->npts, sp.as<int2>(), sd.as<int64_t>(),
                                f->buf.as<double>(), 0, (int64_t)pcs.size(), words, prows, st);
    }
    SG_CUDA(cudaStreamSynchronize(st));  // the piece lists are reused by the next call on this thread
    return SG_OK;
  }
  if (mapped) {
    thread_local DevBuf scratch;
    const size_t need = (size_t)nruns * 2 * sizeof(int64_t);
    if (scratch.bytes < need || scratch.device != f->device) scratch.alloc(f->device, std::max<size_t>(need, 4096));
    cudaStream_t st = as_stream(stream);
    SG_CUDA(cudaMemcpyAsync(scratch.ptr, runs, need, cudaMemcpyHostToDevice, st));
    const unsigned grid = (unsigned)std::min<int64_t>(nruns, 148 * 8);
    copy_runs_kernel<<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(at.devicePointer), f->buf.as<uint32_t>(),
                                           scratch.as<int64_t>(), nruns, (int64_t)(row_bytes / 4));
    SG_CUDA_LAUNCH();
    // the runs were read from pageable memory synchronously; the scratch stays valid until the
    // next call on this thread, which orders after this one on the same stream or syncs
    SG_CUDA(cudaStreamSynchronize(st));
    return SG_OK;
  }
  for (int64_t r = 0; r < nruns; ++r)
    copy_rows(f, runs[2 * r], runs[2 * r + 1], static_cast<const char*>(host) + (size_t)runs[2 * r] * row_bytes,
              nullptr, stream);
  SG_API_END
}

int32_t sg_field_d2h_rows(uint64_t field, int64_t row0, int64_t nrows, void* host, uint64_t stream) {
  SG_API_BEGIN
  Field* f = get<Field>(field, ObjKind::Field);
  SG_REQUIRE(host || nrows == 0, "null host pointer");
  copy_rows(f, row0, nrows, nullptr, host, stream);
  SG_API_END
}

// ---- pinned host memory and device events (timing on the launching stream) ----------------
namespace {
struct Event : Object {
  Event() : Object(ObjKind::Event) {}
  int device = 0;
  cudaEvent_t ev = nullptr;
  ~Event() override {
    if (ev) cudaEventDestroy(ev);
  }
};
}  // namespace

}  // extern "C"

// raw event of a registry handle (runtime.cu: cross-stream waits)
cudaEvent_t sg_event_raw(uint64_t h) { return get<Event>(h, ObjKind::Event)->ev; }

extern "C" {

int32_t sg_host_alloc(size_t bytes, uint64_t* out_ptr) { return sg_host_alloc_flags(bytes, 0, out_ptr); }

// flags bit 0: write-combined (fast CPU writes and PCIe reads, very slow CPU reads)
// flags bit 1: zero-filled (np.zeros semantics) — the current device writes the zeros through
//              the mapped alias over PCIe, no host CPU time
int32_t sg_host_alloc_flags(size_t bytes, int32_t flags, uint64_t* out_ptr) {
  SG_API_BEGIN
  SG_REQUIRE(out_ptr, "null out pointer");
  void* p = nullptr;
  if (!(flags & 1) && bytes >= kMmapPinBytes && (p = mmap_pinned(bytes)) != nullptr) {
    *out_ptr = reinterpret_cast<uint64_t>(p);  // zero-filled by the kernel
    return SG_OK;
  }
  unsigned int f = cudaHostAllocPortable | cudaHostAllocMapped | ((flags & 1) ? cudaHostAllocWriteCombined : 0);
  SG_CUDA(cudaHostAlloc(&p, std::max<size_t>(bytes, 1), f));
  if (flags & 2) {
    void* dp = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dp, p, 0);
    if (e == cudaSuccess) e = cudaMemset(dp, 0, std::max<size_t>(bytes, 1));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      cudaFreeHost(p);
      SG_CUDA(e);
    }
  }
  *out_ptr = reinterpret_cast<uint64_t>(p);
  SG_API_END
}

int32_t sg_host_free(uint64_t ptr) {
  SG_API_BEGIN
  size_t mm = 0;
  {
    std::lock_guard<std::mutex> lk(g_mm_mu);
    auto it = g_mm.find(ptr);
    if (it != g_mm.end()) {
      mm = it->second;
      g_mm.erase(it);
    }
  }
  if (mm) {
    SG_CUDA(cudaHostUnregister(reinterpret_cast<void*>(ptr)));
    munmap(reinterpret_cast<void*>(ptr), mm);
  } else {
    SG_CUDA(cudaFreeHost(reinterpret_cast<void*>(ptr)));
  }
  SG_API_END
}

// Page-lock an existing host range (e.g. a numpy array) so h2d/d2h from it run at full PCIe
// rate and asynchronously; sg_host_unregister undoes it.
int32_t sg_host_register(uint64_t ptr, size_t bytes) {
  SG_API_BEGIN
  SG_REQUIRE(ptr && bytes, "empty range");
  SG_CUDA(cudaHostRegister(reinterpret_cast<void*>(ptr), bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  SG_API_END
}

int32_t sg_host_unregister(uint64_t ptr) {
  SG_API_BEGIN
  SG_CUDA(cudaHostUnregister(reinterpret_cast<void*>(ptr)));
  SG_API_END
}

int32_t sg_event_create(int32_t device, uint64_t* out_event) {
  SG_API_BEGIN
  SG_REQUIRE(out_event, "null out pointer");
  DeviceScope ds(device);
  auto e = std::make_unique<Event>();
  e->device = device;
  SG_CUDA(cudaEventCreate(&e->ev));
  *out_event = registry_put(e.release());
  SG_API_END
}

int32_t sg_event_record(uint64_t event, uint64_t stream) {
  SG_API_BEGIN
  Event* e = get<Event>(event, ObjKind::Event);
  DeviceScope ds(e->device);
  SG_CUDA(cudaEventRecord(e->ev, as_stream(stream)));
  SG_API_END
}

int32_t sg_event_elapsed_ms(uint64_t start, uint64_t end, float* out_ms) {
  SG_API_BEGIN
  Event* a = get<Event>(start, ObjKind::Event);
  Event* b = get<Event>(end, ObjKind::Event);
  SG_REQUIRE(out_ms, "null out pointer");
  DeviceScope ds(b->device);
  SG_CUDA(cudaEventSynchronize(b->ev));
  SG_CUDA(cudaEventElapsedTime(out_ms, a->ev, b->ev));
  SG_API_END
}

}  // extern "C"
