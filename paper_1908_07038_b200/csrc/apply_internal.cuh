// Shared between the apply kernels (apply.cu) and the host-buffer pipeline (execute_host.cu).
#pragma once
#include <vector>

#include "stencil.cuh"

namespace sg {
namespace detail {

constexpr int kMaxFields = 8;

struct ApplyArgs {
  const int4* idx;
  const double4* w;
  int64_t t0, t1;  // target range (positions in `list` when a list is given)
  const int32_t* list;  // optional target list: target = list[position]
  int32_t k;       // stencil points: 3 (FE triangles) or 4 (structured bilinear)
  int32_t levels;
  int32_t nfields;
  const double* src[kMaxFields];
  double* dst[kMaxFields];
  int64_t src_pitch[kMaxFields];
  int64_t dst_pitch[kMaxFields];
};

struct FieldPairs {
  std::vector<Field*> src, dst;
  int32_t levels = -1;
};

// Validates field pairs against the stencil (ShapeMismatch messages of interp.py:208-217).
FieldPairs check_pairs(const Stencil* s, const uint64_t* src_fields, const uint64_t* dst_fields, int nfields);
// Kernel arguments for targets [t0, t1) of up to kMaxFields field pairs starting at f0.
ApplyArgs make_args(const Stencil* s, const FieldPairs& p, int f0, int64_t t0, int64_t t1);
// Chooses and launches the apply kernel for `variant`.
void launch_apply(ApplyArgs a, int variant, cudaStream_t st);

// GPU gather of row pieces out of pinned, mapped host memory (execute_host.cu): piece p =
// (first host row, rows) -> device rows from pdst[p]; rows of `levels` doubles, dense.
// cp.async.bulk copies through a shared-memory ring; pieces of <= gather_piece_rows rows.
int gather_piece_rows(int levels);
bool gather_fits(int levels);
void launch_gather_tma(const double* host, int64_t host_rows, const int2* pieces, const int64_t* pdst, double* out,
                       int64_t p0, int64_t p1, int levels, int piece_rows, cudaStream_t st, int ctas_per_sm = 2);

}  // namespace detail
}  // namespace sg
