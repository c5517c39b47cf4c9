/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into or called by the product
 * (paper_1908_07038_b200/); only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker.
 *
 * Plain-C restatement of the reference's MeshLocator.locate
 * (/root/reference/pkg/src/spheregrid/interp.py:74-117), candidate order and all:
 *   - k nearest mesh nodes of p, k = 8 then 32 (interp.py:30-31, 106), exact brute force,
 *     ordered by squared distance then node index (cKDTree.query order, interp.py:92);
 *   - candidate elements = incident elements of those nodes in ascending element id, first
 *     seen first (interp.py:82-85, 94-100);
 *   - per element its triangles (quads split at the lowest local index, mesh.py:395-403);
 *   - SphericalTriangle raises DegenerateTriangle when |(a x b).c| <= 1e-15 (interp.py:40-43);
 *   - score = min of the signed tests (a x b).p, (b x c).p, (c x a).p (interp.py:46-51) with
 *     np.cross as unfused mul/sub and np.dot as OpenBLAS ddot = fma(c2,p2,fma(c1,p1,c0*p0))
 *     (re-probed on the GPU-box host: tools/host_probe.py);
 *   - keep if score >= -1e-12 and strictly greater than the best so far (interp.py:113).
 * Built with -ffp-contract=off so the compiler cannot fuse the restated arithmetic.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double x, y, z;
} v3;

static v3 ld(const double* xyz, int64_t i) {
  v3 r = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return r;
}
static v3 cross_np(v3 a, v3 b) {
  v3 r;
  r.x = a.y * b.z - a.z * b.y;
  r.y = a.z * b.x - a.x * b.z;
  r.z = a.x * b.y - a.y * b.x;
  return r;
}
static double dot_blas(v3 c, v3 p) { return fma(c.z, p.z, fma(c.y, p.y, c.x * p.x)); }

/* split quads / copy triangles; returns number of triangles written (1 or 2) */
static int element_tris(const int64_t* off, const int64_t* idx, int64_t e, int64_t out[2][3]) {
  int64_t k = off[e + 1] - off[e];
  const int64_t* r = idx + off[e];
  if (k == 3) {
    out[0][0] = r[0]; out[0][1] = r[1]; out[0][2] = r[2];
    return 1;
  }
  int m = 0;
  for (int i = 1; i < 4; ++i)
    if (r[i] < r[m]) m = i;
  int64_t c[4];
  for (int i = 0; i < 4; ++i) c[i] = r[(m + i) % 4];
  out[0][0] = c[0]; out[0][1] = c[1]; out[0][2] = c[2];
  out[1][0] = c[0]; out[1][1] = c[2]; out[1][2] = c[3];
  return 2;
}

/*
 * For each point: out_elem (-1 not located, -2 DegenerateTriangle), out_corners (3 local ids).
 */
int oracle_locate(const double* xyz, int64_t n, const int64_t* off, const int64_t* idx, int64_t nelem,
                  const double* pts, int64_t m, int64_t* out_elem, int64_t* out_corners) {
  /* incidence lists in ascending element id */
  int64_t* cnt = calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < nelem; ++e)
    for (int64_t i = off[e]; i < off[e + 1]; ++i) cnt[idx[i] + 1]++;
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  int64_t* inc = malloc(sizeof(int64_t) * (size_t)(cnt[n] > 0 ? cnt[n] : 1));
  int64_t* fill = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  memcpy(fill, cnt, sizeof(int64_t) * (size_t)n);
  for (int64_t e = 0; e < nelem; ++e)
    for (int64_t i = off[e]; i < off[e + 1]; ++i) inc[fill[idx[i]]++] = e;
  unsigned char* seen = calloc((size_t)(nelem > 0 ? nelem : 1), 1);
  int64_t* cand = malloc(sizeof(int64_t) * (size_t)(nelem > 0 ? nelem : 1));
  for (int64_t t = 0; t < m; ++t) {
    v3 p = ld(pts, t);
    out_elem[t] = -1;
    const int ks[2] = {8, 32};
    int done = 0;
    for (int pass = 0; pass < 2 && !done; ++pass) {
      int k = ks[pass] < n ? ks[pass] : (int)n;
      double bd[32];
      int64_t bi[32];
      int nb = 0;
      for (int64_t i = 0; i < n; ++i) {
        double dx = xyz[3 * i] - p.x, dy = xyz[3 * i + 1] - p.y, dz = xyz[3 * i + 2] - p.z;
        double d = dx * dx + dy * dy + dz * dz;
        if (nb < k || d < bd[nb - 1]) {
          int j = nb < k ? nb++ : nb - 1;
          while (j > 0 && bd[j - 1] > d) {
            bd[j] = bd[j - 1];
            bi[j] = bi[j - 1];
            --j;
          }
          bd[j] = d;
          bi[j] = i;
        }
      }
      int64_t nc = 0;
      for (int a = 0; a < nb; ++a)
        for (int64_t q = cnt[bi[a]]; q < cnt[bi[a] + 1]; ++q) {
          int64_t e = inc[q];
          if (!seen[e]) {
            seen[e] = 1;
            cand[nc++] = e;
          }
        }
      int have = 0;
      double best = 0.0;
      for (int64_t c = 0; c < nc && out_elem[t] != -2; ++c) {
        int64_t tr[2][3];
        int nt = element_tris(off, idx, cand[c], tr);
        for (int s = 0; s < nt; ++s) {
          v3 a = ld(xyz, tr[s][0]), b = ld(xyz, tr[s][1]), cc = ld(xyz, tr[s][2]);
          v3 ab = cross_np(a, b);
          if (fabs(dot_blas(ab, cc)) <= 1e-15) {
            out_elem[t] = -2;
            break;
          }
          double t1 = dot_blas(ab, p), t2 = dot_blas(cross_np(b, cc), p), t3 = dot_blas(cross_np(cc, a), p);
          double score = t1;
          if (t2 < score) score = t2;
          if (t3 < score) score = t3;
          if (score >= -1e-12 && (!have || score > best)) {
            have = 1;
            best = score;
            out_elem[t] = cand[c];
            out_corners[3 * t] = tr[s][0];
            out_corners[3 * t + 1] = tr[s][1];
            out_corners[3 * t + 2] = tr[s][2];
          }
        }
      }
      for (int64_t c = 0; c < nc; ++c) seen[cand[c]] = 0;
      if (have || out_elem[t] == -2) done = 1;
    }
    if (out_elem[t] == -1) out_corners[3 * t] = out_corners[3 * t + 1] = out_corners[3 * t + 2] = -1;
  }
  free(cnt);
  free(inc);
  free(fill);
  free(seen);
  free(cand);
  return 0;
}

/*
 * Same scoring, with the candidate nodes supplied: knn[t*k .. t*k+k) are the k nearest mesh
 * nodes of point t in cKDTree order (interp.py:92 — the caller runs the reference's own
 * scipy cKDTree query).  Incidence lists are built once per call.  out_elem: -1 not located
 * among these candidates, -2 DegenerateTriangle.
 */
int oracle_locate_knn(const double* xyz, int64_t n, const int64_t* off, const int64_t* idx, int64_t nelem,
                      const double* pts, int64_t m, const int64_t* knn, int k, int64_t* out_elem,
                      int64_t* out_corners) {
  int64_t* cnt = calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < nelem; ++e)
    for (int64_t i = off[e]; i < off[e + 1]; ++i) cnt[idx[i] + 1]++;
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  int64_t* inc = malloc(sizeof(int64_t) * (size_t)(cnt[n] > 0 ? cnt[n] : 1));
  int64_t* fill = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  memcpy(fill, cnt, sizeof(int64_t) * (size_t)n);
  for (int64_t e = 0; e < nelem; ++e)
    for (int64_t i = off[e]; i < off[e + 1]; ++i) inc[fill[idx[i]]++] = e;
  for (int64_t t = 0; t < m; ++t) {
    v3 p = ld(pts, t);
    out_elem[t] = -1;
    out_corners[3 * t] = out_corners[3 * t + 1] = out_corners[3 * t + 2] = -1;
    int64_t cand[4096];
    int nc = 0;
    for (int a = 0; a < k; ++a) {
      const int64_t node = knn[t * k + a];
      if (node < 0 || node >= n) continue;
      for (int64_t q = cnt[node]; q < cnt[node + 1]; ++q) {
        int64_t e = inc[q];
        int dup = 0;
        for (int j = 0; j < nc; ++j)
          if (cand[j] == e) { dup = 1; break; }
        if (!dup && nc < 4096) cand[nc++] = e;
      }
    }
    int have = 0;
    double best = 0.0;
    for (int c = 0; c < nc && out_elem[t] != -2; ++c) {
      int64_t tr[2][3];
      int nt = element_tris(off, idx, cand[c], tr);
      for (int s = 0; s < nt; ++s) {
        v3 a = ld(xyz, tr[s][0]), b = ld(xyz, tr[s][1]), cc = ld(xyz, tr[s][2]);
        v3 ab = cross_np(a, b);
        if (fabs(dot_blas(ab, cc)) <= 1e-15) {
          out_elem[t] = -2;
          break;
        }
        double t1 = dot_blas(ab, p), t2 = dot_blas(cross_np(b, cc), p), t3 = dot_blas(cross_np(cc, a), p);
        double score = t1;
        if (t2 < score) score = t2;
        if (t3 < score) score = t3;
        if (score >= -1e-12 && (!have || score > best)) {
          have = 1;
          best = score;
          out_elem[t] = cand[c];
          out_corners[3 * t] = tr[s][0];
          out_corners[3 * t + 1] = tr[s][1];
          out_corners[3 * t + 2] = tr[s][2];
        }
      }
    }
  }
  free(cnt);
  free(inc);
  free(fill);
  return 0;
}

/* np.linalg.solve(M, p) for 3x3 systems restated operation for operation as numpy's bundled
 * OpenBLAS dgesv evaluates it (getrf_single -> getf2 left-looking LU, getrs -> dlaswp + trsv):
 * the kernels' roundings — dot / dgemv_n tail sums as FMA chains from 0 subtracted as one
 * term, pivot scaling by the reciprocal, FMA axpy in trsv, division by the diagonal.  The
 * checker for the device's lu_solve3 (csrc/locate.cu); pinned bitwise against np.linalg.solve
 * and the golden weights by tests/test_oracle.py.  M row-major (m, 3, 3); returns 0, or the
 * 1-based index of the first singular system. */
int64_t oracle_dgesv3(const double* Mall, const double* pall, double* xall, int64_t m) {
  int64_t bad = 0;
  for (int64_t t = 0; t < m; ++t) {
    const double* Mi = Mall + 9 * t;
    double A[3][3]; /* column-major: A[col][row] */
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) A[j][i] = Mi[3 * i + j];
    int ipiv[3], singular = 0;
    for (int j = 0; j < 3; ++j) {
      double* b = A[j];
      for (int i = 0; i < j; ++i)
        if (ipiv[i] != i) { double s = b[i]; b[i] = b[ipiv[i]]; b[ipiv[i]] = s; }
      for (int i = 1; i < j; ++i) {
        double d = 0.0;
        for (int k = 0; k < i; ++k) d = fma(A[k][i], b[k], d);
        b[i] = b[i] - d;
      }
      for (int i = j; i < 3; ++i) {
        double s = 0.0;
        for (int k = 0; k < j; ++k) s = fma(A[k][i], b[k], s);
        b[i] = fma(-1.0, s, b[i]);
      }
      int jp = j;
      for (int i = j + 1; i < 3; ++i)
        if (fabs(b[i]) > fabs(b[jp])) jp = i;
      ipiv[j] = jp;
      const double piv = b[jp];
      if (piv == 0.0) { singular = 1; continue; }
      if (jp != j)
        for (int k = 0; k <= j; ++k) { double s = A[k][j]; A[k][j] = A[k][jp]; A[k][jp] = s; }
      const double r = 1.0 / piv;
      for (int i = j + 1; i < 3; ++i) b[i] = b[i] * r;
    }
    double* y = xall + 3 * t;
    y[0] = pall[3 * t]; y[1] = pall[3 * t + 1]; y[2] = pall[3 * t + 2];
    if (singular) { if (!bad) bad = t + 1; continue; }
    for (int i = 0; i < 3; ++i)
      if (ipiv[i] != i) { double s = y[i]; y[i] = y[ipiv[i]]; y[ipiv[i]] = s; }
    for (int i = 0; i < 3; ++i)
      for (int k = i + 1; k < 3; ++k) y[k] = fma(-y[i], A[i][k], y[k]);
    for (int i = 2; i >= 0; --i) {
      y[i] = y[i] / A[i][i];
      for (int k = 0; k < i; ++k) y[k] = fma(-y[i], A[i][k], y[k]);
    }
  }
  return bad;
}
