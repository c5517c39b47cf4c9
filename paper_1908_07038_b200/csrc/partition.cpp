// Native matching partition: PointCloudIndex.query + matching_partition (partition.py:53-88).
//
// For every target point: the nearest master grid point (poles excluded, partition.py:59),
// with near-equal distances (d <= best*(1+1e-12), partition.py:15, 62-75) resolved to the
// smallest global index.  Distances are recomputed like np.linalg.norm(xyz - p, axis=1):
// sqrt((dx*dx + dy*dy) + dz*dz) with separately rounded operations (built with
// -ffp-contract=off).  Instead of a kd-tree the search uses the master grid's row
// structure: rows are scanned outward from the target's latitude while the chord lower bound
// 2 sin(|Δφ|/2) can still reach the tie window; inside a row the 4 points around the
// target's longitude are candidates (a row's nearest point is one of its two lon
// neighbours).
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "sg_internal.h"

namespace {

constexpr double kTieRtol = 1e-12;  // partition.py:15

struct Master {
  int32_t nrows;
  std::vector<double> lat;  // radians, north -> south (descending)
  std::vector<int64_t> nlon, off;
  const double* xyz;
};

inline double dist_np(const double* a, const double* p) {
  const double dx = a[0] - p[0], dy = a[1] - p[1], dz = a[2] - p[2];
  const double sx = dx * dx, sy = dy * dy, sz = dz * dz;
  return std::sqrt((sx + sy) + sz);
}

int64_t nearest_one(const Master& M, const double* p) {
  const double phi = std::asin(std::max(-1.0, std::min(1.0, p[2])));
  double lam = std::atan2(p[1], p[0]);
  if (lam < 0) lam += 2 * M_PI;
  // first row with lat <= phi (lat descending)
  int64_t lo = 0, hi = M.nrows;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (M.lat[mid] > phi) lo = mid + 1; else hi = mid;
  }
  struct Cand { double d; int64_t g; };
  Cand cands[256];
  int nc = 0;
  double best = INFINITY;
  auto scan_row = [&](int64_t j) {
    const int64_t n = M.nlon[j];
    const double step = 2 * M_PI / (double)n;
    int64_t i0 = (int64_t)std::floor(lam / step);
    const int64_t span = std::min<int64_t>(n, 4);
    for (int64_t k = 0; k < span; ++k) {
      int64_t i = ((i0 - 1 + k) % n + n) % n;
      const int64_t g = M.off[j] + i;
      const double d = dist_np(M.xyz + 3 * g, p);
      if (nc < 256) cands[nc++] = Cand{d, g};
      if (d < best) best = d;
    }
  };
  auto lower_bound_row = [&](int64_t j) { return 2.0 * std::sin(0.5 * std::fabs(M.lat[j] - phi)); };
  const int64_t jn = std::min<int64_t>(std::max<int64_t>(lo - 1, 0), M.nrows - 1);  // north of (or at) phi
  const int64_t js = std::min<int64_t>(lo, M.nrows - 1);
  scan_row(jn);
  if (js != jn) scan_row(js);
  for (int64_t j = jn - 1; j >= 0; --j) {
    if (lower_bound_row(j) * (1.0 - 1e-9) > best * (1.0 + 1e-11) + 1e-300) break;
    scan_row(j);
  }
  for (int64_t j = js + 1; j < M.nrows; ++j) {
    if (lower_bound_row(j) * (1.0 - 1e-9) > best * (1.0 + 1e-11) + 1e-300) break;
    scan_row(j);
  }
  const double lim = best * (1.0 + kTieRtol);
  int64_t g = INT64_MAX;
  for (int i = 0; i < nc; ++i)
    if (cands[i].d <= lim && cands[i].g < g) g = cands[i].g;
  return g;
}

}  // namespace

extern "C" int32_t sg_matching_partition(int32_t nrows, const double* master_lat_deg, const int64_t* master_nlons,
                                         const double* master_xyz, const double* target_xyz, int64_t m,
                                         int32_t nthreads, int64_t* out_index) {
  SG_API_BEGIN
  SG_REQUIRE(nrows >= 1 && master_lat_deg && master_nlons && master_xyz, "bad master grid");
  SG_REQUIRE(m == 0 || (target_xyz && out_index), "null target arrays");
  Master M;
  M.nrows = nrows;
  M.xyz = master_xyz;
  M.off.assign(nrows + 1, 0);
  for (int32_t j = 0; j < nrows; ++j) {
    M.lat.push_back(master_lat_deg[j] * (M_PI / 180.0));
    M.nlon.push_back(master_nlons[j]);
    M.off[j + 1] = M.off[j] + master_nlons[j];
  }
  int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, m / 1024));
  std::vector<std::thread> pool;
  for (int w = 0; w < nt; ++w)
    pool.emplace_back([&, w]() {
      for (int64_t k = w; k < m; k += nt) out_index[k] = nearest_one(M, target_xyz + 3 * k);
    });
  for (auto& t : pool) t.join();
  SG_API_END
}
