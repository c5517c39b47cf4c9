// Device stencil of InterpolationWeights (interp.py:120-133): per target the three local
// source node indices (int32, padded to an int4 for one 16-B load) and the three weights
// (padded to 4 doubles, two 16-B loads).  48 B per target in HBM; the algorithmic 36 B
// (int32 indices + fp64 weights) is what the roofline counts.
#pragma once
#include "cuda_util.cuh"

namespace sg {

struct Stencil : Object {
  Stencil() : Object(ObjKind::Stencil) {}
  int device = 0;
  int64_t m = 0;
  int32_t k = 3;                 // points per target: 3 (FE) or 4 (structured bilinear)
  int64_t source_nnodes = 0;
  int64_t distinct_sources = 0;  // U: distinct source rows referenced
  DevBuf idx;                    // int4[m]
  DevBuf w;                      // double4[m]
  void* host_plan = nullptr;     // pipelined host-buffer execute plan (apply.cu)
  void destroy_host_plan();
  ~Stencil() override { destroy_host_plan(); }
};

// Builds the device arrays from device-resident int32 index / fp64 weight k-tuples
// (idx/w are [m][s->k] on the device) and counts distinct referenced source rows.
void stencil_finalize(Stencil* s, const int32_t* d_idx3, const double* d_w3, cudaStream_t st);

}  // namespace sg
