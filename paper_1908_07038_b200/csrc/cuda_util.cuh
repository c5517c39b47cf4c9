// CUDA helpers shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>

#include "sg_internal.h"

#define SG_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      sg::throw_error(SG_DOMAIN_ERROR, "CudaError: %s failed: %s (%s:%d)", #call,      \
                      cudaGetErrorString(_e), __FILE__, __LINE__);                     \
  } while (0)

#define SG_CUDA_LAUNCH() SG_CUDA(cudaGetLastError())

namespace sg {

inline cudaStream_t as_stream(uint64_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Sets the calling thread's device for the scope of one API call.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    SG_CUDA(cudaGetDevice(&prev));
    if (prev != dev) SG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceScope() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

// Device allocation owned by a registry object.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int device = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void alloc(int dev, size_t n) {
    free();
    device = dev;
    bytes = n;
    if (n) SG_CUDA(cudaMalloc(&ptr, n));
  }
  void free() {
    if (ptr) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (cur != device) cudaSetDevice(device);
      cudaFree(ptr);
      if (cur != device && cur >= 0) cudaSetDevice(cur);
    }
    ptr = nullptr;
    bytes = 0;
  }
  ~DevBuf() { free(); }
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

// Pitched (npts, levels) field storage: Field.device of the reference (field.py:102).
struct Field : Object {
  Field() : Object(ObjKind::Field) {}
  int device = 0;
  int64_t npts = 0;
  int32_t levels = 0;
  int32_t itemsize = 8;
  int64_t pitch = 0;  // elements
  DevBuf buf;
};

// Row pitch policy: dense rows (pitch == levels), exactly the reference host layout.
// Measured (profiles/, round 1): with 128-B padded rows every gathered 1096-B row cost 1152 B
// of DRAM reads (HBM fetches 64-B granules), 5% over the algorithmic bytes; dense rows let
// the boundary granule of two neighbouring source points — which neighbouring targets read
// together — be fetched once, and make h2d/d2h plain contiguous copies at full PCIe rate.
inline int64_t field_pitch_elems(int32_t levels, int32_t /*itemsize*/) { return levels; }

}  // namespace sg
