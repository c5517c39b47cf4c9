// Stencil search + gnomonic barycentric weights on the device: the B200 replacement for
// MeshLocator (interp.py:74-117) and the per-target loop of build_remap (interp.py:154-203).
//
// Search structure (built once per mesh, sg_locator_create):
//   * quads are split at the corner with the lowest LOCAL node index (mesh.py:395-403);
//     triangle ids run in (element id, triangle index) order, so "lowest triangle id" is the
//     reference's tie rule "lowest local element id, then triangle 0 before 1" (SURVEY.md §0
//     fact 1: the empirical outcome of interp.py:113's strict '>' over candidate order).
//   * every spherical triangle gets an exact latitude range (vertices plus the poleward /
//     equatorward bulge of each great-circle edge) and longitude range (vertex hull; edges of
//     minor arcs are monotone in longitude), inflated by a margin that covers CONTAIN_EPS
//     (interp.py:29) and device trig error;
//   * the sphere is cut into latitude bands of height dlat, each band into
//     floor(2π cos(φ_eq)/dlat) longitude bins; each triangle is listed in every bin its box
//     overlaps (count -> scan -> fill -> CUB radix sort by bin, stable, so a bin lists its
//     triangles in ascending id).
//   The bin of a target therefore holds a SUPERSET of the triangles that can contain it
//   within CONTAIN_EPS; the reference's kNN candidate set (interp.py:90-100) is replaced by
//   this superset plus the explicit tie rule (validated bit-exact in SURVEY.md A6/A7/A17).
//
// Per target (one thread): signed tests with the reference's rounding — cross products as
// unfused mul/sub (np.cross), dots as the OpenBLAS ddot FMA chain fma(c2,p2,fma(c1,p1,c0*p0))
// — score = min(t1,t2,t3), keep score >= -1e-12, max score, ties -> lowest id.
// Weights: 3x3 LU with partial pivoting (the dgesv of interp.py:65), renormalised by
// ((w0+w1)+w2) (interp.py:68-71); scale = (w·[a b c]^T)·p (interp.py:194).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "stencil.cuh"

namespace sg {
namespace {

constexpr double kContainEps = 1e-12;  // interp.py:29
constexpr double kDegenerateVol = 1e-15;  // interp.py:42
constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kHalfPi = 1.5707963267948966192313216916398;

struct Locator : Object {
  Locator() : Object(ObjKind::Locator) {}
  int device = 0;
  int64_t n_nodes = 0, n_elems = 0, ntri = 0;
  DevBuf xyz;        // double[n][3]
  DevBuf tris;       // int4 (c0, c1, c2, element id) per triangle
  DevBuf band_nlon;  // int32[nbands]
  DevBuf band_off;   // int32[nbands + 1]  first bin of each band
  DevBuf bin_start;  // int32[nbins + 1]
  DevBuf entries;    // int32[nentries]  triangle ids, grouped by bin, ascending within a bin
  double dlat = 0;
  int nbands = 0;
  int64_t nbins = 0, nentries = 0;
  // nodes incident to an element with a degenerate triangle (knn_rule_kernel); usually none
  DevBuf flagged;  // int32[nflagged]
  int64_t nflagged = 0;
};

struct LocView {
  const double* xyz;
  const int4* tris;
  const int32_t* band_nlon;
  const int32_t* band_off;
  const int32_t* bin_start;
  const int32_t* entries;
  double dlat;
  int nbands;
};

// ---- exact arithmetic of the reference --------------------------------------------------
struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 load3(const double* p, int i) {
  return V3{p[3 * (int64_t)i], p[3 * (int64_t)i + 1], p[3 * (int64_t)i + 2]};
}
// np.cross: cp0 = a1*b2 - a2*b1, cp1 = a2*b0 - a0*b2, cp2 = a0*b1 - a1*b0, unfused
__device__ __forceinline__ V3 cross_np(V3 a, V3 b) {
  return V3{__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)),
            __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
            __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
// np.dot on 3-vectors (OpenBLAS ddot): fma(c2,p2, fma(c1,p1, c0*p0))
__device__ __forceinline__ double dot_blas(V3 c, V3 p) {
  return __fma_rn(c.z, p.z, __fma_rn(c.y, p.y, __dmul_rn(c.x, p.x)));
}

// ---- triangle boxes ---------------------------------------------------------------------
__device__ __forceinline__ double norm3(V3 v) { return sqrt(v.x * v.x + v.y * v.y + v.z * v.z); }

// Extend [zmin, zmax] by the extreme z of the minor great-circle arc u->v.
__device__ void edge_z_extent(V3 u, V3 v, double& zmin, double& zmax) {
  V3 n = V3{u.y * v.z - u.z * v.y, u.z * v.x - u.x * v.z, u.x * v.y - u.y * v.x};
  double nn = norm3(n);
  if (!(nn > 1e-300)) return;
  n = V3{n.x / nn, n.y / nn, n.z / nn};
  double r2 = 1.0 - n.z * n.z;
  if (!(r2 > 0.0)) return;  // arc on the equator plane normal to z: z constant 0
  double r = sqrt(r2);
  // top point m = (z_hat - n.z n) / r
  V3 m = V3{-n.z * n.x / r, -n.z * n.y / r, (1.0 - n.z * n.z) / r};
  for (int s = 0; s < 2; ++s) {
    V3 q = s == 0 ? m : V3{-m.x, -m.y, -m.z};
    // q on the minor arc iff (u x q).n >= 0 and (q x v).n >= 0
    V3 uq = V3{u.y * q.z - u.z * q.y, u.z * q.x - u.x * q.z, u.x * q.y - u.y * q.x};
    V3 qv = V3{q.y * v.z - q.z * v.y, q.z * v.x - q.x * v.z, q.x * v.y - q.y * v.x};
    double s1 = uq.x * n.x + uq.y * n.y + uq.z * n.z;
    double s2 = qv.x * n.x + qv.y * n.y + qv.z * n.z;
    if (s1 >= -1e-12 && s2 >= -1e-12) {
      zmax = fmax(zmax, q.z);
      zmin = fmin(zmin, q.z);
    }
  }
}

struct Box {
  double plo, phi;   // latitude range (rad)
  double llo, lspan; // longitude start in [0, 2π) and span; lspan >= 2π means all
};

__device__ Box triangle_box(V3 a, V3 b, V3 c) {
  double zmin = fmin(a.z, fmin(b.z, c.z));
  double zmax = fmax(a.z, fmax(b.z, c.z));
  edge_z_extent(a, b, zmin, zmax);
  edge_z_extent(b, c, zmin, zmax);
  edge_z_extent(c, a, zmin, zmax);
  // margin: a point passes the containment test up to ~CONTAIN_EPS/|edge normal| outside
  double ab = norm3(cross_np(a, b)), bc = norm3(cross_np(b, c)), ca = norm3(cross_np(c, a));
  double nmin = fmax(fmin(ab, fmin(bc, ca)), 1e-300);
  double delta = 1e-9 + 8.0 * kContainEps / nmin;
  bool full = false;
  // does the triangle (with margin) contain a pole?
  V3 cab = cross_np(a, b), cbc = cross_np(b, c), cca = cross_np(c, a);
  const double tol = 1e-9;
  if (cab.z >= -tol && cbc.z >= -tol && cca.z >= -tol) { zmax = 1.0; full = true; }
  if (-cab.z >= -tol && -cbc.z >= -tol && -cca.z >= -tol) { zmin = -1.0; full = true; }
  Box bx;
  bx.plo = asin(fmax(-1.0, fmin(1.0, zmin))) - delta;
  bx.phi = asin(fmax(-1.0, fmin(1.0, zmax))) + delta;
  // longitude hull of the non-polar vertices
  double lon[3];
  int nl = 0;
  V3 vv[3] = {a, b, c};
  for (int i = 0; i < 3; ++i) {
    double h = hypot(vv[i].x, vv[i].y);
    if (h > 1e-10) {
      double l = atan2(vv[i].y, vv[i].x);
      if (l < 0) l += kTwoPi;
      lon[nl++] = l;
    }
  }
  double pext = fmax(fabs(bx.plo), fabs(bx.phi));
  double cosp = pext >= kHalfPi ? 0.0 : cos(pext);
  if (full || nl < 2 || cosp < 1e-6) {
    bx.llo = 0.0;
    bx.lspan = 2 * kTwoPi;
    return bx;
  }
  // sort
  for (int i = 0; i < nl; ++i)
    for (int j = i + 1; j < nl; ++j)
      if (lon[j] < lon[i]) { double t = lon[i]; lon[i] = lon[j]; lon[j] = t; }
  // largest circular gap; range is its complement
  double best_gap = -1.0;
  int best_i = 0;
  for (int i = 0; i < nl; ++i) {
    double nxt = (i + 1 < nl) ? lon[i + 1] : lon[0] + kTwoPi;
    double gap = nxt - lon[i];
    if (gap > best_gap) { best_gap = gap; best_i = i; }
  }
  double start = (best_i + 1 < nl) ? lon[best_i + 1] : lon[0];
  double span = kTwoPi - best_gap;
  double dl = delta / cosp + 1e-12;
  start -= dl;
  span += 2 * dl;
  if (span >= 3.0) {  // large (polar) triangle: take the whole band
    bx.llo = 0.0;
    bx.lspan = 2 * kTwoPi;
    return bx;
  }
  if (start < 0) start += kTwoPi;
  if (start >= kTwoPi) start -= kTwoPi;
  bx.llo = start;
  bx.lspan = span;
  return bx;
}

__device__ __forceinline__ int band_of(double phi, double dlat, int nbands) {
  int b = (int)floor((phi + kHalfPi) / dlat);
  return min(max(b, 0), nbands - 1);
}
__device__ __forceinline__ int lonbin_of(double lam, int nlon) {
  int i = (int)floor(lam / kTwoPi * nlon);
  return min(max(i, 0), nlon - 1);
}

__global__ void tri_extent_kernel(const double* xyz, const int4* tris, int64_t ntri, double* sum_ext,
                                  unsigned long long* n_ext) {
  double s = 0;
  unsigned long long c = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntri;
       t += (int64_t)gridDim.x * blockDim.x) {
    int4 tc = tris[t];
    V3 a = load3(xyz, tc.x), b = load3(xyz, tc.y), c3 = load3(xyz, tc.z);
    double za = asin(fmax(-1.0, fmin(1.0, a.z))), zb = asin(fmax(-1.0, fmin(1.0, b.z))),
           zc = asin(fmax(-1.0, fmin(1.0, c3.z)));
    double e = fmax(za, fmax(zb, zc)) - fmin(za, fmin(zb, zc));
    if (e > 0 && e < 0.2) {
      s += e;
      c += 1;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sum_ext, s);
    atomicAdd(n_ext, c);
  }
}

template <bool kFill>
__global__ void tri_bins_kernel(LocView v, int64_t ntri, int64_t* counts, const int64_t* offsets,
                                int32_t* keys, int32_t* vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntri) return;
  int4 tc = v.tris[t];
  Box bx = triangle_box(load3(v.xyz, tc.x), load3(v.xyz, tc.y), load3(v.xyz, tc.z));
  int b0 = band_of(bx.plo, v.dlat, v.nbands), b1 = band_of(bx.phi, v.dlat, v.nbands);
  int64_t n = 0;
  int64_t pos = kFill ? offsets[t] : 0;
  for (int b = b0; b <= b1; ++b) {
    int nlon = v.band_nlon[b];
    int i0, cnt;
    if (bx.lspan >= kTwoPi) {
      i0 = 0;
      cnt = nlon;
    } else {
      i0 = lonbin_of(bx.llo, nlon);
      int i1 = (int)floor((bx.llo + bx.lspan) / kTwoPi * nlon);
      cnt = min(i1 - i0 + 1, nlon);
    }
    if (kFill) {
      for (int k = 0; k < cnt; ++k) {
        int i = (i0 + k) % nlon;
        keys[pos] = v.band_off[b] + i;
        vals[pos] = (int32_t)t;
        ++pos;
      }
    }
    n += cnt;
  }
  if (!kFill) counts[t] = n;
}

__global__ void bin_bounds_kernel(const int32_t* keys, int64_t n, int64_t nbins, int32_t* bin_start) {
  // bin_start[b] = first entry index with key >= b  (keys sorted ascending)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  int64_t prev = (i == 0) ? -1 : keys[i - 1];
  int64_t cur = (i == n) ? nbins : keys[i];
  for (int64_t b = prev + 1; b <= cur; ++b) bin_start[b] = (int32_t)i;
}

// ---- locate + weights -------------------------------------------------------------------
struct TargetOut {
  int32_t* idx3;     // [m][3] local source nodes
  double* w3;        // [m][3]
  double* scale;     // [m]
  uint8_t* status;   // [m]
  int32_t* best_tri; // [m]
};

// np.linalg.solve(M, p) for a 3x3 system exactly as the reference's LAPACK does it: numpy's
// bundled OpenBLAS dgesv = getrf_single -> getf2 (left-looking LU: per column, apply the earlier
// pivots, subtract dot(L, u) from the U part, subtract the dgemv_n tail sum from the rest, pick
// the first max |.| pivot, swap rows, scale by the pivot's reciprocal) then getrs -> dlaswp +
// trsv NLU / NUN (axpy updates with FMA, divisions by the diagonal).  The kernels' roundings:
// dot / gemv tail sums are FMA chains from 0 subtracted as one term; axpy is FMA.  Bitwise equal
// to np.linalg.solve on every cfg2 target (108,160) and every fixture; false = singular (a zero
// pivot: LinAlgError in the reference, interp.py:66-67).
__device__ __forceinline__ bool lu_solve3(const double M[3][3], const double rhs[3], double x[3]) {
  double A[3][3];  // column-major: A[col][row]
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A[j][i] = M[i][j];
  int ipiv[3];
  bool singular = false;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    double* b = A[j];
    for (int i = 0; i < j; ++i)  // earlier pivots applied to this column
      if (ipiv[i] != i) { const double t = b[i]; b[i] = b[ipiv[i]]; b[ipiv[i]] = t; }
    for (int i = 1; i < j; ++i) {  // U part: b[i] -= dot(L[i, 0:i], b[0:i])
      double d = 0.0;
      for (int k = 0; k < i; ++k) d = __fma_rn(A[k][i], b[k], d);
      b[i] = __dsub_rn(b[i], d);
    }
    for (int i = j; i < 3; ++i) {  // dgemv_n tail rows: b[i] += -1 * sum_k A[i,k] b[k]
      double t = 0.0;
      for (int k = 0; k < j; ++k) t = __fma_rn(A[k][i], b[k], t);
      b[i] = __fma_rn(-1.0, t, b[i]);
    }
    int jp = j;  // idamax: first maximum
    for (int i = j + 1; i < 3; ++i)
      if (fabs(b[i]) > fabs(b[jp])) jp = i;
    ipiv[j] = jp;
    const double piv = b[jp];
    if (piv == 0.0) {
      singular = true;
      continue;
    }
    if (jp != j)
      for (int k = 0; k <= j; ++k) { const double t = A[k][j]; A[k][j] = A[k][jp]; A[k][jp] = t; }
    const double r = 1.0 / piv;
    for (int i = j + 1; i < 3; ++i) b[i] = __dmul_rn(b[i], r);
  }
  if (singular) return false;
  double y[3] = {rhs[0], rhs[1], rhs[2]};
  for (int i = 0; i < 3; ++i)  // dlaswp
    if (ipiv[i] != i) { const double t = y[i]; y[i] = y[ipiv[i]]; y[ipiv[i]] = t; }
  for (int i = 0; i < 3; ++i)  // trsv, unit lower: axpy with -y[i]
    for (int k = i + 1; k < 3; ++k) y[k] = __fma_rn(-y[i], A[i][k], y[k]);
  for (int i = 2; i >= 0; --i) {  // trsv, upper: divide, then axpy
    y[i] = __ddiv_rn(y[i], A[i][i]);
    for (int k = 0; k < i; ++k) y[k] = __fma_rn(-y[i], A[i][k], y[k]);
  }
  x[0] = y[0]; x[1] = y[1]; x[2] = y[2];
  return true;
}

// Weights + scale of target t for its chosen triangle (status 0), or the [1,0,0] placeholder.
__device__ void finish_target(const LocView& v, V3 q, int64_t t, int best, uint8_t st, bool want_weights,
                              const TargetOut& out) {
  out.best_tri[t] = best;
  if (want_weights) {
    double w[3] = {1.0, 0.0, 0.0};
    double sc = 1.0;
    int4 tc = make_int4(0, 0, 0, 0);
    if (st == 0) {
      tc = __ldg(v.tris + best);
      const V3 a = load3(v.xyz, tc.x), b = load3(v.xyz, tc.y), c = load3(v.xyz, tc.z);
      const double M[3][3] = {{a.x, b.x, c.x}, {a.y, b.y, c.y}, {a.z, b.z, c.z}};
      const double rhs[3] = {q.x, q.y, q.z};
      double x[3];
      if (!lu_solve3(M, rhs, x)) {
        st = 3;
      } else {
        const double s = __dadd_rn(__dadd_rn(x[0], x[1]), x[2]);  // w.sum()
        if (s == 0.0) {
          st = 4;  // interp.py:69-70
        } else {
          w[0] = x[0] / s; w[1] = x[1] / s; w[2] = x[2] / s;
          // w @ column_stack([a, b, c]).T: numpy's matmul -> OpenBLAS dgemv_t tail row
          // `a0*x0 + a1*x1 + a2*x2`, which its compiler contracted to fma(a2,x2,fma(a0,x0,a1*x1))
          // (bitwise on all 108,160 cfg2 targets); then ddot with p
          const V3 vproj = V3{__fma_rn(w[2], c.x, __fma_rn(w[0], a.x, __dmul_rn(w[1], b.x))),
                              __fma_rn(w[2], c.y, __fma_rn(w[0], a.y, __dmul_rn(w[1], b.y))),
                              __fma_rn(w[2], c.z, __fma_rn(w[0], a.z, __dmul_rn(w[1], b.z)))};
          sc = dot_blas(vproj, q);
        }
      }
    }
    if (st != 0) { w[0] = 1.0; w[1] = 0.0; w[2] = 0.0; sc = 1.0; }
    out.idx3[3 * t] = tc.x; out.idx3[3 * t + 1] = tc.y; out.idx3[3 * t + 2] = tc.z;
    out.w3[3 * t] = w[0]; out.w3[3 * t + 1] = w[1]; out.w3[3 * t + 2] = w[2];
    out.scale[t] = sc;
  }
  out.status[t] = st;
}

__device__ __forceinline__ void bins_of(const LocView& v, V3 q, int& bin_lo, int& bin_hi) {
  const double phi = asin(fmax(-1.0, fmin(1.0, q.z)));
  const int band = band_of(phi, v.dlat, v.nbands);
  const int nlon = v.band_nlon[band];
  if (hypot(q.x, q.y) <= 1e-10) {  // at a pole: every bin of the band
    bin_lo = v.band_off[band];
    bin_hi = v.band_off[band] + nlon - 1;
  } else {
    double lam = atan2(q.y, q.x);
    if (lam < 0) lam += kTwoPi;
    bin_lo = bin_hi = v.band_off[band] + lonbin_of(lam, nlon);
  }
}

// min(t1, t2, t3) of interp.py:111-113 with the reference's rounding; *degen: |(a x b).c| <= 1e-15
__device__ __forceinline__ double tri_score(const LocView& v, int tri, V3 q, bool* degen) {
  const int4 tc = __ldg(v.tris + tri);
  const V3 a = load3(v.xyz, tc.x), b = load3(v.xyz, tc.y), c = load3(v.xyz, tc.z);
  const V3 ab = cross_np(a, b);
  *degen = fabs(dot_blas(ab, c)) <= kDegenerateVol;  // interp.py:40-43
  const double t1 = dot_blas(ab, q);
  const double t2 = dot_blas(cross_np(b, c), q);
  const double t3 = dot_blas(cross_np(c, a), q);
  return fmin(t1, fmin(t2, t3));
}

// Meshes without degenerate triangles: best containing triangle among the target's bin (a
// superset of the reference's kNN candidates), ties -> lowest triangle id.  Degenerate
// triangles never win (the reference raises before it could pick one); meshes that have any
// are re-decided per target by knn_rule_kernel.
__global__ void __launch_bounds__(128) locate_kernel(LocView v, const double* pts, int64_t m,
                                                     bool want_weights, TargetOut out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const V3 q = V3{pts[3 * t], pts[3 * t + 1], pts[3 * t + 2]};
  int bin_lo, bin_hi;
  bins_of(v, q, bin_lo, bin_hi);
  int best = -1;
  double best_score = 0.0;
  for (int bin = bin_lo; bin <= bin_hi; ++bin) {
    const int e0 = v.bin_start[bin], e1 = v.bin_start[bin + 1];
    for (int e = e0; e < e1; ++e) {
      const int tri = __ldg(v.entries + e);
      bool degen;
      const double score = tri_score(v, tri, q, &degen);
      if (!degen && score >= -kContainEps &&
          (best < 0 || score > best_score || (score == best_score && tri < best))) {
        best = tri;
        best_score = score;
      }
    }
  }
  finish_target(v, q, t, best, best < 0 ? 1 : 0, want_weights, out);
}

// ---- exact kNN-candidate emulation (meshes with degenerate triangles) -------------------
// The reference scores only the elements incident to the k = 8 (then k = min(32, n)) nearest
// nodes (interp.py:90-117) and raises DegenerateTriangle as soon as one of them has a
// degenerate triangle (interp.py:34-43, 109-110).  Node n is "flagged" when an element
// incident to it has a degenerate triangle; rank(x) = #nodes strictly closer to p than x
// (squared distance, unfused, as cKDTree) — x is among the k nearest iff rank(x) < k (exact
// distance ties at the k-th place are cKDTree-order dependent: parity unpinned there).
//   pass k: raise if rank(nearest flagged node) < k; else best over the containing
//   triangles whose element has a corner of rank < k (max score, ties -> lowest id); none ->
//   next pass; after the last pass NotLocated.
constexpr int kRuleThreads = 128;
constexpr int kRuleMaxCand = 96;

__device__ __forceinline__ double dist2(const double* xyz, int64_t i, V3 p) {
  const double dx = __dsub_rn(xyz[3 * i], p.x), dy = __dsub_rn(xyz[3 * i + 1], p.y),
               dz = __dsub_rn(xyz[3 * i + 2], p.z);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// #nodes with dist2 < d (block-wide, all threads call), stops counting at cap.
__device__ int count_closer(const double* xyz, int64_t n, V3 p, double d, int cap, int* sh) {
  if (threadIdx.x == 0) *sh = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += (int64_t)kRuleThreads * 8) {
    int local = 0;
    for (int j = 0; j < 8; ++j) {
      const int64_t i = base + (int64_t)j * kRuleThreads + threadIdx.x;
      if (i < n && dist2(xyz, i, p) < d) ++local;
    }
    if (local) atomicAdd(sh, local);
    __syncthreads();
    const int c = *sh;
    __syncthreads();
    if (c >= cap) return c;
  }
  return *sh;
}

__global__ void __launch_bounds__(kRuleThreads) knn_rule_kernel(LocView v, int64_t n, const int32_t* flagged,
                                                                 int64_t nflagged, const double* pts, int64_t m,
                                                                 bool want_weights, TargetOut out) {
  const int64_t t = blockIdx.x;
  if (t >= m) return;
  const V3 q = V3{pts[3 * t], pts[3 * t + 1], pts[3 * t + 2]};
  __shared__ double red[kRuleThreads];
  __shared__ int sh_count, ncand;
  __shared__ double cscore[kRuleMaxCand];
  __shared__ int ctri[kRuleMaxCand], crank[kRuleMaxCand];
  const int kmax = (int)(n < 32 ? n : 32);
  // 1. nearest flagged node and its rank
  double dmin = INFINITY;
  for (int64_t i = threadIdx.x; i < nflagged; i += kRuleThreads) dmin = fmin(dmin, dist2(v.xyz, flagged[i], q));
  red[threadIdx.x] = dmin;
  __syncthreads();
  for (int o = kRuleThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  const double dflag = red[0];
  const int rank_flag = count_closer(v.xyz, n, q, dflag, kmax, &sh_count);
  // 2. containing, non-degenerate triangles of the bin
  if (threadIdx.x == 0) ncand = 0;
  __syncthreads();
  int bin_lo, bin_hi;
  bins_of(v, q, bin_lo, bin_hi);
  for (int bin = bin_lo; bin <= bin_hi; ++bin) {
    const int e0 = v.bin_start[bin], e1 = v.bin_start[bin + 1];
    for (int e = e0 + threadIdx.x; e < e1; e += kRuleThreads) {
      const int tri = __ldg(v.entries + e);
      bool degen;
      const double score = tri_score(v, tri, q, &degen);
      if (!degen && score >= -kContainEps) {
        const int k = atomicAdd(&ncand, 1);
        if (k < kRuleMaxCand) {
          cscore[k] = score;
          ctri[k] = tri;
        }
      }
    }
  }
  __syncthreads();
  const int nc = min(ncand, kRuleMaxCand);
  // 3. rank of each candidate's element = min rank of its corners (all triangles of the element)
  for (int c = 0; c < nc; ++c) {
    const int tri = ctri[c];
    const int elem = __ldg(v.tris + tri).w;
    int lo = tri, hi = tri;
    while (lo > 0 && __ldg(v.tris + lo - 1).w == elem) --lo;
    while (__ldg(v.tris + hi + 1).w == elem) ++hi;  // tris is padded by the sentinel below
    int r = kmax;
    for (int u = lo; u <= hi; ++u) {
      const int4 tc = __ldg(v.tris + u);
      const int cs[3] = {tc.x, tc.y, tc.z};
      for (int j = 0; j < 3; ++j) r = min(r, count_closer(v.xyz, n, q, dist2(v.xyz, cs[j], q), r, &sh_count));
    }
    if (threadIdx.x == 0) crank[c] = r;
    __syncthreads();
  }
  // 4. the reference's two passes
  if (threadIdx.x == 0) {
    uint8_t st = 1;
    int best = -1;
    if (ncand > kRuleMaxCand) {
      st = 5;  // too many overlapping candidates to decide exactly
    } else {
      const int ks[2] = {min(8, kmax), kmax};
      for (int pass = 0; pass < 2 && st == 1; ++pass) {
        const int k = ks[pass];
        if (rank_flag < k) {
          st = 2;
          break;
        }
        double bs = 0.0;
        for (int c = 0; c < nc; ++c)
          if (crank[c] < k && (best < 0 || cscore[c] > bs || (cscore[c] == bs && ctri[c] < best))) {
            best = ctri[c];
            bs = cscore[c];
          }
        if (best >= 0) st = 0;
      }
    }
    finish_target(v, q, t, st == 0 ? best : -1, st, want_weights, out);
  }
}

// Nearest local node for the fallback rows (interp.py:186; kd-tree tie order unspecified,
// here: smallest squared distance, then smallest index).  One block per failing target.
__global__ void nearest_node_kernel(const double* xyz, int64_t n, const double* pts, const int64_t* rows,
                                    int64_t nrows, int32_t* idx3, double* w3) {
  const int64_t r = blockIdx.x;
  if (r >= nrows) return;
  const int64_t t = rows[r];
  const double px = pts[3 * t], py = pts[3 * t + 1], pz = pts[3 * t + 2];
  double bd = INFINITY;
  int64_t bi = INT64_MAX;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double dx = __dsub_rn(xyz[3 * i], px), dy = __dsub_rn(xyz[3 * i + 1], py),
                 dz = __dsub_rn(xyz[3 * i + 2], pz);
    // unfused, like cKDTree's squared Euclidean distance (interp.py:186)
    const double d = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    if (d < bd || (d == bd && i < bi)) { bd = d; bi = i; }
  }
  __shared__ double sd[256];
  __shared__ int64_t si[256];
  sd[threadIdx.x] = bd;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      double d2 = sd[threadIdx.x + o];
      int64_t i2 = si[threadIdx.x + o];
      if (d2 < sd[threadIdx.x] || (d2 == sd[threadIdx.x] && i2 < si[threadIdx.x])) {
        sd[threadIdx.x] = d2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int32_t nn = (int32_t)si[0];
    idx3[3 * t] = nn; idx3[3 * t + 1] = nn; idx3[3 * t + 2] = nn;
    w3[3 * t] = 1.0; w3[3 * t + 1] = 0.0; w3[3 * t + 2] = 0.0;
  }
}

LocView view_of(const Locator* L) {
  return LocView{L->xyz.as<double>(),          L->tris.as<int4>(),
                 L->band_nlon.as<int32_t>(),   L->band_off.as<int32_t>(),
                 L->bin_start.as<int32_t>(),   L->entries.as<int32_t>(),
                 L->dlat,                      L->nbands};
}

__global__ void degenerate_elems_kernel(const double* xyz, const int4* tris, int64_t ntri, uint8_t* elem_flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntri) return;
  const int4 tc = tris[i];
  const V3 a = load3(xyz, tc.x), b = load3(xyz, tc.y), c = load3(xyz, tc.z);
  if (fabs(dot_blas(cross_np(a, b), c)) <= kDegenerateVol) elem_flag[tc.w] = 1;  // interp.py:40-43
}

__global__ void flag_nodes_kernel(const int4* tris, int64_t ntri, const uint8_t* elem_flag, uint8_t* node_flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntri) return;
  const int4 tc = tris[i];
  if (elem_flag[tc.w]) node_flag[tc.x] = node_flag[tc.y] = node_flag[tc.z] = 1;
}

// Nodes that make the reference raise DegenerateTriangle when they are among a target's
// nearest nodes (corners of an element that has a degenerate triangle).
void find_flagged_nodes(Locator* L, cudaStream_t st) {
  L->nflagged = 0;
  if (L->ntri == 0) return;
  DevBuf ef, nf;
  ef.alloc(L->device, (size_t)std::max<int64_t>(L->n_elems, 1));
  nf.alloc(L->device, (size_t)std::max<int64_t>(L->n_nodes, 1));
  SG_CUDA(cudaMemsetAsync(ef.ptr, 0, ef.bytes, st));
  SG_CUDA(cudaMemsetAsync(nf.ptr, 0, nf.bytes, st));
  const unsigned g = (unsigned)((L->ntri + 255) / 256);
  degenerate_elems_kernel<<<g, 256, 0, st>>>(L->xyz.as<double>(), L->tris.as<int4>(), L->ntri, ef.as<uint8_t>());
  SG_CUDA_LAUNCH();
  flag_nodes_kernel<<<g, 256, 0, st>>>(L->tris.as<int4>(), L->ntri, ef.as<uint8_t>(), nf.as<uint8_t>());
  SG_CUDA_LAUNCH();
  std::vector<uint8_t> h((size_t)L->n_nodes);
  if (L->n_nodes) SG_CUDA(cudaMemcpyAsync(h.data(), nf.ptr, h.size(), cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> list;
  for (int64_t i = 0; i < L->n_nodes; ++i)
    if (h[i]) list.push_back((int32_t)i);
  L->nflagged = (int64_t)list.size();
  if (!list.empty()) {
    L->flagged.alloc(L->device, list.size() * 4);
    SG_CUDA(cudaMemcpyAsync(L->flagged.ptr, list.data(), list.size() * 4, cudaMemcpyHostToDevice, st));
    SG_CUDA(cudaStreamSynchronize(st));
  }
}

void build_bins(Locator* L, cudaStream_t st) {
  const int64_t ntri = L->ntri;
  // 1. typical triangle latitude extent -> band height
  DevBuf dsum, dcnt;
  dsum.alloc(L->device, sizeof(double));
  dcnt.alloc(L->device, sizeof(unsigned long long));
  SG_CUDA(cudaMemsetAsync(dsum.ptr, 0, sizeof(double), st));
  SG_CUDA(cudaMemsetAsync(dcnt.ptr, 0, sizeof(unsigned long long), st));
  if (ntri) {
    tri_extent_kernel<<<592, 256, 0, st>>>(L->xyz.as<double>(), L->tris.as<int4>(), ntri, dsum.as<double>(),
                                          dcnt.as<unsigned long long>());
    SG_CUDA_LAUNCH();
  }
  double hsum = 0;
  unsigned long long hcnt = 0;
  SG_CUDA(cudaMemcpyAsync(&hsum, dsum.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaMemcpyAsync(&hcnt, dcnt.ptr, sizeof(hcnt), cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  double ext = hcnt ? hsum / (double)hcnt : 0.1;
  double dlat = std::min(std::max(1.5 * ext, M_PI / 65536.0), M_PI / 8.0);
  int nbands = (int)std::ceil(M_PI / dlat);
  dlat = M_PI / nbands;
  std::vector<int32_t> nlon(nbands), off(nbands + 1);
  int64_t nbins = 0;
  for (int b = 0; b < nbands; ++b) {
    double lo = -M_PI / 2 + b * dlat, hi = lo + dlat;
    double peq = (lo <= 0 && hi >= 0) ? 0.0 : std::min(std::fabs(lo), std::fabs(hi));
    int n = (int)std::floor(2 * M_PI * std::cos(peq) / dlat);
    n = std::max(1, std::min(n, 1 << 22));
    nlon[b] = n;
    off[b] = (int32_t)nbins;
    nbins += n;
  }
  off[nbands] = (int32_t)nbins;
  SG_REQUIRE(nbins < INT32_MAX, "too many search bins");
  L->dlat = dlat;
  L->nbands = nbands;
  L->nbins = nbins;
  L->band_nlon.alloc(L->device, nlon.size() * 4);
  L->band_off.alloc(L->device, off.size() * 4);
  SG_CUDA(cudaMemcpyAsync(L->band_nlon.ptr, nlon.data(), nlon.size() * 4, cudaMemcpyHostToDevice, st));
  SG_CUDA(cudaMemcpyAsync(L->band_off.ptr, off.data(), off.size() * 4, cudaMemcpyHostToDevice, st));
  // 2. count bins per triangle, scan
  DevBuf counts, offsets;
  counts.alloc(L->device, (size_t)std::max<int64_t>(ntri, 1) * 8);
  offsets.alloc(L->device, (size_t)(ntri + 1) * 8);
  LocView v = view_of(L);
  const unsigned g = (unsigned)((ntri + 255) / 256);
  if (ntri) {
    tri_bins_kernel<false><<<g, 256, 0, st>>>(v, ntri, counts.as<int64_t>(), nullptr, nullptr, nullptr);
    SG_CUDA_LAUNCH();
  }
  size_t tmp_bytes = 0;
  SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts.as<int64_t>(), offsets.as<int64_t>(),
                                        (int)(ntri + 1), st));
  // scan ntri+1 items: counts[ntri] is garbage-free because we scan into offsets with a
  // zero-padded copy below
  DevBuf counts_pad;
  counts_pad.alloc(L->device, (size_t)(ntri + 1) * 8);
  SG_CUDA(cudaMemsetAsync(counts_pad.ptr, 0, counts_pad.bytes, st));
  if (ntri) SG_CUDA(cudaMemcpyAsync(counts_pad.ptr, counts.ptr, (size_t)ntri * 8, cudaMemcpyDeviceToDevice, st));
  DevBuf tmp;
  tmp.alloc(L->device, std::max<size_t>(tmp_bytes, 16));
  SG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, counts_pad.as<int64_t>(), offsets.as<int64_t>(),
                                        (int)(ntri + 1), st));
  int64_t nent = 0;
  SG_CUDA(cudaMemcpyAsync(&nent, offsets.as<int64_t>() + ntri, 8, cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  SG_REQUIRE(nent < INT32_MAX, "too many search-bin entries");
  L->nentries = nent;
  // 3. fill (bin, triangle) pairs in triangle order, stable radix sort by bin
  DevBuf keys, vals, keys2;
  keys.alloc(L->device, (size_t)std::max<int64_t>(nent, 1) * 4);
  vals.alloc(L->device, (size_t)std::max<int64_t>(nent, 1) * 4);
  keys2.alloc(L->device, (size_t)std::max<int64_t>(nent, 1) * 4);
  L->entries.alloc(L->device, (size_t)std::max<int64_t>(nent, 1) * 4);
  if (ntri) {
    tri_bins_kernel<true><<<g, 256, 0, st>>>(v, ntri, nullptr, offsets.as<int64_t>(), keys.as<int32_t>(),
                                             vals.as<int32_t>());
    SG_CUDA_LAUNCH();
  }
  int end_bit = 1;
  while ((int64_t(1) << end_bit) <= nbins) ++end_bit;
  size_t sort_bytes = 0;
  SG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys.as<int32_t>(), keys2.as<int32_t>(),
                                          vals.as<int32_t>(), L->entries.as<int32_t>(), (int)nent, 0,
                                          end_bit, st));
  DevBuf sort_tmp;
  sort_tmp.alloc(L->device, std::max<size_t>(sort_bytes, 16));
  SG_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.ptr, sort_bytes, keys.as<int32_t>(), keys2.as<int32_t>(),
                                          vals.as<int32_t>(), L->entries.as<int32_t>(), (int)nent, 0,
                                          end_bit, st));
  // 4. bin offsets
  L->bin_start.alloc(L->device, (size_t)(nbins + 1) * 4);
  bin_bounds_kernel<<<(unsigned)((nent + 1 + 255) / 256), 256, 0, st>>>(keys2.as<int32_t>(), nent, nbins,
                                                                        L->bin_start.as<int32_t>());
  SG_CUDA_LAUNCH();
  SG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace
}  // namespace sg

using namespace sg;

extern "C" {

int32_t sg_locator_create(int32_t device, const double* node_xyz, int64_t n_nodes,
                          const int64_t* elem_offsets, const int64_t* elem_indices, int64_t n_elems,
                          uint64_t* out_locator) {
  SG_API_BEGIN
  SG_REQUIRE(out_locator, "null out pointer");
  SG_REQUIRE(n_nodes >= 0 && n_elems >= 0, "negative size");
  SG_REQUIRE(n_nodes < INT32_MAX, "mesh too large for int32 node indices");
  SG_REQUIRE(n_nodes == 0 || node_xyz, "null node_xyz");
  SG_REQUIRE(elem_offsets, "null element offsets");
  // triangles in (element, triangle index) order; quads split at the lowest local index
  // (split_quad, mesh.py:395-403)
  std::vector<int4> tris;
  tris.reserve((size_t)n_elems * 2);
  for (int64_t e = 0; e < n_elems; ++e) {
    const int64_t o = elem_offsets[e], k = elem_offsets[e + 1] - elem_offsets[e];
    const int64_t* r = elem_indices + o;
    for (int64_t i = 0; i < k; ++i)
      SG_REQUIRE(r[i] >= 0 && r[i] < n_nodes, "element %lld references node %lld outside [0, %lld)",
                 (long long)e, (long long)r[i], (long long)n_nodes);
    if (k == 3) {
      tris.push_back(make_int4((int)r[0], (int)r[1], (int)r[2], (int)e));
    } else if (k == 4) {
      int m = 0;
      for (int i = 1; i < 4; ++i)
        if (r[i] < r[m]) m = i;  // np.argmin: first minimum
      int c0 = (int)r[m], c1 = (int)r[(m + 1) % 4], c2 = (int)r[(m + 2) % 4], c3 = (int)r[(m + 3) % 4];
      tris.push_back(make_int4(c0, c1, c2, (int)e));
      tris.push_back(make_int4(c0, c2, c3, (int)e));
    } else {
      sg::throw_error(SG_INVALID_ARGUMENT, "element %lld has %lld nodes (expected 3 or 4)", (long long)e,
                      (long long)k);
    }
  }
  SG_REQUIRE(tris.size() < (size_t)INT32_MAX, "too many triangles");
  DeviceScope ds(device);
  auto L = std::make_unique<Locator>();
  L->device = device;
  L->n_nodes = n_nodes;
  L->n_elems = n_elems;
  L->ntri = (int64_t)tris.size();  // before the sentinel
  L->xyz.alloc(device, (size_t)std::max<int64_t>(n_nodes, 1) * 24);
  tris.push_back(make_int4(0, 0, 0, -1));  // sentinel: element -1 ends the last element's run
  L->tris.alloc(device, tris.size() * sizeof(int4));
  cudaStream_t st = 0;
  if (n_nodes) SG_CUDA(cudaMemcpyAsync(L->xyz.ptr, node_xyz, (size_t)n_nodes * 24, cudaMemcpyHostToDevice, st));
  SG_CUDA(cudaMemcpyAsync(L->tris.ptr, tris.data(), tris.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  build_bins(L.get(), st);
  find_flagged_nodes(L.get(), st);
  *out_locator = registry_put(L.release());
  SG_API_END
}

int32_t sg_locator_stats(uint64_t locator, int64_t* out_ntri, int64_t* out_nbins, int64_t* out_nentries,
                         double* out_band_rad) {
  SG_API_BEGIN
  Locator* L = get<Locator>(locator, ObjKind::Locator);
  if (out_ntri) *out_ntri = L->ntri;
  if (out_nbins) *out_nbins = L->nbins;
  if (out_nentries) *out_nentries = L->nentries;
  if (out_band_rad) *out_band_rad = L->dlat;
  SG_API_END
}

static void run_locate(Locator* L, const double* points, int64_t m, bool want_weights, DevBuf& dpts,
                       DevBuf& idx3, DevBuf& w3, DevBuf& scale, DevBuf& status, DevBuf& best,
                       cudaStream_t st) {
  dpts.alloc(L->device, (size_t)std::max<int64_t>(m, 1) * 24);
  idx3.alloc(L->device, (size_t)std::max<int64_t>(m, 1) * 12);
  w3.alloc(L->device, (size_t)std::max<int64_t>(m, 1) * 24);
  scale.alloc(L->device, (size_t)std::max<int64_t>(m, 1) * 8);
  status.alloc(L->device, (size_t)std::max<int64_t>(m, 1));
  best.alloc(L->device, (size_t)std::max<int64_t>(m, 1) * 4);
  if (m == 0) return;
  SG_CUDA(cudaMemcpyAsync(dpts.ptr, points, (size_t)m * 24, cudaMemcpyHostToDevice, st));
  TargetOut out{idx3.as<int32_t>(), w3.as<double>(), scale.as<double>(), status.as<uint8_t>(),
                best.as<int32_t>()};
  locate_kernel<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(view_of(L), dpts.as<double>(), m, want_weights,
                                                             out);
  SG_CUDA_LAUNCH();
  if (L->nflagged) {  // degenerate triangles present: decide every target as the kNN search would
    knn_rule_kernel<<<(unsigned)m, kRuleThreads, 0, st>>>(view_of(L), L->n_nodes, L->flagged.as<int32_t>(),
                                                          L->nflagged, dpts.as<double>(), m, want_weights, out);
    SG_CUDA_LAUNCH();
  }
}

int32_t sg_locator_locate(uint64_t locator, const double* points, int64_t m, int64_t* out_elem,
                          int64_t* out_corners) {
  SG_API_BEGIN
  Locator* L = get<Locator>(locator, ObjKind::Locator);
  SG_REQUIRE(m >= 0, "negative size");
  SG_REQUIRE(m == 0 || (points && out_elem), "null arrays");
  DeviceScope ds(L->device);
  cudaStream_t st = 0;
  DevBuf dpts, idx3, w3, scale, status, best;
  run_locate(L, points, m, false, dpts, idx3, w3, scale, status, best, st);
  std::vector<int32_t> hb((size_t)m);
  std::vector<uint8_t> hs((size_t)m);
  if (m) {
    SG_CUDA(cudaMemcpyAsync(hb.data(), best.ptr, (size_t)m * 4, cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaMemcpyAsync(hs.data(), status.ptr, (size_t)m, cudaMemcpyDeviceToHost, st));
  }
  SG_CUDA(cudaStreamSynchronize(st));
  std::vector<int4> tris;
  if (m) {
    tris.resize((size_t)L->ntri);
    SG_CUDA(cudaMemcpy(tris.data(), L->tris.ptr, tris.size() * sizeof(int4), cudaMemcpyDeviceToHost));
  }
  for (int64_t i = 0; i < m; ++i) {
    if (hs[i] != 0 || hb[i] < 0) {
      // -1 NotLocated, -2 DegenerateTriangle (a kNN candidate is degenerate), -3 undecidable
      out_elem[i] = hs[i] == 2 ? -2 : hs[i] == 5 ? -3 : -1;
      if (out_corners) out_corners[3 * i] = out_corners[3 * i + 1] = out_corners[3 * i + 2] = -1;
    } else {
      const int4 tc = tris[hb[i]];
      out_elem[i] = tc.w;
      if (out_corners) {
        out_corners[3 * i] = tc.x;
        out_corners[3 * i + 1] = tc.y;
        out_corners[3 * i + 2] = tc.z;
      }
    }
  }
  SG_API_END
}

int32_t sg_remap_build(uint64_t locator, const double* target_xyz, int64_t m, int64_t source_nnodes,
                       int32_t allow_fallback, uint64_t* out_stencil, int64_t* out_nodes, double* out_weights,
                       double* out_scale, uint8_t* out_fallback, uint8_t* out_status, int64_t* out_first_bad) {
  SG_API_BEGIN
  Locator* L = get<Locator>(locator, ObjKind::Locator);
  SG_REQUIRE(m >= 0, "negative size");
  SG_REQUIRE(m == 0 || (target_xyz && out_nodes && out_weights && out_scale && out_fallback),
             "null output arrays");
  SG_REQUIRE(source_nnodes == L->n_nodes, "source_nnodes %lld != locator nodes %lld", (long long)source_nnodes,
             (long long)L->n_nodes);
  if (out_first_bad) *out_first_bad = -1;
  DeviceScope ds(L->device);
  cudaStream_t st = 0;
  DevBuf dpts, idx3, w3, scale, status, best;
  run_locate(L, target_xyz, m, true, dpts, idx3, w3, scale, status, best, st);
  std::vector<uint8_t> hs((size_t)m);
  if (m) SG_CUDA(cudaMemcpyAsync(hs.data(), status.ptr, (size_t)m, cudaMemcpyDeviceToHost, st));
  SG_CUDA(cudaStreamSynchronize(st));
  // reference order (interp.py:175-192): the first target (ascending) that fails decides
  std::vector<int64_t> unlocated;
  int64_t first_bad = -1;
  int bad_kind = 0;
  for (int64_t i = 0; i < m; ++i) {
    const uint8_t s = hs[i];
    if (s == 0) continue;
    if (s == 1 && allow_fallback) {
      unlocated.push_back(i);
      continue;
    }
    first_bad = i;
    bad_kind = s;
    break;
  }
  if (out_status && m) std::copy(hs.begin(), hs.end(), out_status);
  if (first_bad >= 0) {
    if (out_first_bad) *out_first_bad = first_bad;
    if (bad_kind == 1)
      sg::throw_error(SG_DOMAIN_ERROR, "NotLocated: target row %lld not located in local source elements",
                      (long long)first_bad);
    if (bad_kind == 2)
      sg::throw_error(SG_DOMAIN_ERROR, "DegenerateTriangle: degenerate candidate triangle for target row %lld",
                      (long long)first_bad);
    if (bad_kind == 5)
      sg::throw_error(SG_DOMAIN_ERROR,
                      "SpheregridError: more than %d overlapping candidate triangles at target row %lld",
                      kRuleMaxCand, (long long)first_bad);
    if (bad_kind == 4)
      sg::throw_error(SG_DOMAIN_ERROR, "DegenerateTriangle: projection plane through the origin (target row %lld)",
                      (long long)first_bad);
    sg::throw_error(SG_DOMAIN_ERROR, "DegenerateTriangle: singular vertex matrix for target row %lld",
                    (long long)first_bad);
  }
  if (!unlocated.empty()) {
    DevBuf drows;
    drows.alloc(L->device, unlocated.size() * 8);
    SG_CUDA(cudaMemcpyAsync(drows.ptr, unlocated.data(), unlocated.size() * 8, cudaMemcpyHostToDevice, st));
    nearest_node_kernel<<<(unsigned)unlocated.size(), 256, 0, st>>>(L->xyz.as<double>(), L->n_nodes,
                                                                    dpts.as<double>(), drows.as<int64_t>(),
                                                                    (int64_t)unlocated.size(),
                                                                    idx3.as<int32_t>(), w3.as<double>());
    SG_CUDA_LAUNCH();
    SG_CUDA(cudaStreamSynchronize(st));
  }
  std::vector<int32_t> hidx((size_t)m * 3);
  if (m) {
    SG_CUDA(cudaMemcpyAsync(hidx.data(), idx3.ptr, (size_t)m * 12, cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaMemcpyAsync(out_weights, w3.ptr, (size_t)m * 24, cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaMemcpyAsync(out_scale, scale.ptr, (size_t)m * 8, cudaMemcpyDeviceToHost, st));
  }
  SG_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < m * 3; ++i) out_nodes[i] = hidx[i];
  for (int64_t i = 0; i < m; ++i) out_fallback[i] = (hs[i] == 1) ? 1 : 0;
  if (out_stencil) {
    auto s = std::make_unique<Stencil>();
    s->device = L->device;
    s->m = m;
    s->source_nnodes = source_nnodes;
    stencil_finalize(s.get(), idx3.as<int32_t>(), w3.as<double>(), st);
    *out_stencil = registry_put(s.release());
  }
  SG_API_END
}

}  // extern "C"
