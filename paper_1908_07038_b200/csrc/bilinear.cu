// Structured-bilinear remap stencils (BASELINE.json configs[4]).
//
// The reference has NO such method (its only operator is the gnomonic triangle remap,
// interp.py:1-12), so this is a written definition, restated on the CPU in
// oracle/oracle.py:bilinear_stencil; parity is against that restatement only ("parity
// unpinned" with respect to the reference).  Definition, for a target at (lon λ, lat φ) in
// degrees on a source grid with rows north -> south (lat_j, n_j points at 360·i/n_j):
//   * bracketing rows: j = last row with lat_j >= φ; rows (j, j+1); β = (lat_j - φ) /
//     (lat_j - lat_{j+1})
//   * in a row of n points: x = (λ · n) / 360, i = floor(x) (clamped to [0, n-1]),
//     α = x - i, neighbours i and (i+1) mod n
//   * weights  w = [(1-β)(1-α_j), (1-β)α_j, β(1-α_{j+1}), β α_{j+1}]
//   * polar caps (φ above the first / below the last row) use the pole node as a virtual
//     row at ±90° holding both neighbours: w = [1-β, β(1-α), βα, 0] with
//     β = (90 - φ)/(90 - lat_0) (north) or (φ + 90)/(lat_last + 90) (south), nodes
//     [pole, i, i+1, pole]; without pole nodes a cap target is NotLocated.
// Every operation is a single IEEE op in the order written (no FMA), so the device and the
// numpy restatement agree bit for bit.  Nodes are mapped global -> local through the
// mesh's numbering; a node missing from the local (owned + halo) mesh -> NotLocated.
#include <algorithm>
#include <vector>

#include "stencil.cuh"

namespace sg {
namespace {

struct RowGrid {
  const double* lat;     // degrees, descending
  const int64_t* nlon;
  const int64_t* off;
  int nrows;
  int64_t npts;          // grid points; poles (if any) are npts, npts+1
  int has_poles;
  const int32_t* g2l;    // global -> local (-1 absent), size npts + 2
};

__device__ __forceinline__ void row_pair(const RowGrid& g, int j, double lam, int32_t& ia, int32_t& ib,
                                         double& alpha) {
  const int64_t n = g.nlon[j];
  const double x = __ddiv_rn(__dmul_rn(lam, (double)n), 360.0);
  int64_t i = (int64_t)floor(x);
  if (i < 0) i = 0;
  if (i > n - 1) i = n - 1;
  alpha = __dsub_rn(x, (double)i);
  ia = (int32_t)(g.off[j] + i);
  ib = (int32_t)(g.off[j] + (i + 1) % n);
}

__global__ void bilinear_kernel(RowGrid g, const double* lonlat, int64_t m, int32_t* nodes4, double* w4,
                                uint8_t* status) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const double lam = lonlat[2 * t], phi = lonlat[2 * t + 1];
  int32_t gn[4];
  double w[4];
  uint8_t st = 0;
  if (phi > g.lat[0] || phi < g.lat[g.nrows - 1]) {
    const bool north = phi > g.lat[0];
    const int j = north ? 0 : g.nrows - 1;
    if (!g.has_poles) {
      st = 1;
      gn[0] = gn[1] = gn[2] = gn[3] = 0;
      w[0] = 1.0; w[1] = w[2] = w[3] = 0.0;
    } else {
      const int32_t pole = (int32_t)(north ? g.npts : g.npts + 1);
      const double beta = north ? __ddiv_rn(__dsub_rn(90.0, phi), __dsub_rn(90.0, g.lat[0]))
                                : __ddiv_rn(__dadd_rn(phi, 90.0), __dadd_rn(g.lat[j], 90.0));
      double a;
      row_pair(g, j, lam, gn[1], gn[2], a);
      gn[0] = gn[3] = pole;
      w[0] = __dsub_rn(1.0, beta);
      w[1] = __dmul_rn(beta, __dsub_rn(1.0, a));
      w[2] = __dmul_rn(beta, a);
      w[3] = 0.0;
    }
  } else {
    // last row with lat >= phi (rows descending); keep j + 1 inside the grid
    int lo = 0, hi = g.nrows - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (g.lat[mid] >= phi) lo = mid; else hi = mid - 1;
    }
    int j = lo;
    if (j == g.nrows - 1) j = g.nrows - 2;  // phi == lat of the last row
    if (g.nrows < 2) j = 0;
    const double beta = g.nrows < 2 ? 0.0 : __ddiv_rn(__dsub_rn(g.lat[j], phi), __dsub_rn(g.lat[j], g.lat[j + 1]));
    double a0, a1;
    row_pair(g, j, lam, gn[0], gn[1], a0);
    row_pair(g, g.nrows < 2 ? j : j + 1, lam, gn[2], gn[3], a1);
    const double ob = __dsub_rn(1.0, beta);
    w[0] = __dmul_rn(ob, __dsub_rn(1.0, a0));
    w[1] = __dmul_rn(ob, a0);
    w[2] = __dmul_rn(beta, __dsub_rn(1.0, a1));
    w[3] = __dmul_rn(beta, a1);
  }
  for (int k = 0; k < 4; ++k) {
    const int32_t l = g.g2l[gn[k]];
    if (l < 0 && st == 0) st = 1;
    nodes4[4 * t + k] = l < 0 ? 0 : l;
    w4[4 * t + k] = w[k];
  }
  status[t] = st;
}

}  // namespace
}  // namespace sg

using namespace sg;

extern "C" int32_t sg_bilinear_build(int32_t device, int32_t nrows, const double* lat_deg, const int64_t* nlons,
                                     int32_t has_poles, const int64_t* node_global, int64_t n_nodes,
                                     const double* target_lonlat, int64_t m, uint64_t* out_stencil,
                                     int64_t* out_nodes, double* out_weights, uint8_t* out_status,
                                     int64_t* out_first_bad) {
  SG_API_BEGIN
  SG_REQUIRE(nrows >= 1 && lat_deg && nlons, "bad source grid");
  SG_REQUIRE(m >= 0 && n_nodes >= 0 && n_nodes < INT32_MAX, "bad sizes");
  SG_REQUIRE(m == 0 || (target_lonlat && out_nodes && out_weights), "null arrays");
  std::vector<int64_t> off(nrows + 1, 0);
  for (int j = 0; j < nrows; ++j) {
    SG_REQUIRE(nlons[j] >= 1, "row %d has no points", j);
    off[j + 1] = off[j] + nlons[j];
  }
  const int64_t npts = off[nrows];
  std::vector<int32_t> g2l((size_t)npts + 2, -1);
  for (int64_t i = 0; i < n_nodes; ++i) {
    SG_REQUIRE(node_global[i] >= 0 && node_global[i] < npts + 2, "node_global[%lld] out of range", (long long)i);
    g2l[node_global[i]] = (int32_t)i;
  }
  if (out_first_bad) *out_first_bad = -1;
  DeviceScope ds(device);
  cudaStream_t st = 0;
  DevBuf dlat, dnl, doff, dg2l, dll, dnodes, dw, dstat;
  dlat.alloc(device, nrows * 8);
  dnl.alloc(device, nrows * 8);
  doff.alloc(device, (nrows + 1) * 8);
  dg2l.alloc(device, g2l.size() * 4);
  dll.alloc(device, (size_t)std::max<int64_t>(m, 1) * 16);
  dnodes.alloc(device, (size_t)std::max<int64_t>(m, 1) * 16);
  dw.alloc(device, (size_t)std::max<int64_t>(m, 1) * 32);
  dstat.alloc(device, (size_t)std::max<int64_t>(m, 1));
  SG_CUDA(cudaMemcpyAsync(dlat.ptr, lat_deg, nrows * 8, cudaMemcpyHostToDevice, st));
  SG_CUDA(cudaMemcpyAsync(dnl.ptr, nlons, nrows * 8, cudaMemcpyHostToDevice, st));
  SG_CUDA(cudaMemcpyAsync(doff.ptr, off.data(), (nrows + 1) * 8, cudaMemcpyHostToDevice, st));
  SG_CUDA(cudaMemcpyAsync(dg2l.ptr, g2l.data(), g2l.size() * 4, cudaMemcpyHostToDevice, st));
  if (m) {
    SG_CUDA(cudaMemcpyAsync(dll.ptr, target_lonlat, (size_t)m * 16, cudaMemcpyHostToDevice, st));
    RowGrid g{dlat.as<double>(), dnl.as<int64_t>(), doff.as<int64_t>(), nrows, npts, has_poles, dg2l.as<int32_t>()};
    bilinear_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(g, dll.as<double>(), m, dnodes.as<int32_t>(),
                                                                 dw.as<double>(), dstat.as<uint8_t>());
    SG_CUDA_LAUNCH();
  }
  std::vector<int32_t> hn((size_t)m * 4);
  std::vector<uint8_t> hs((size_t)m);
  if (m) {
    SG_CUDA(cudaMemcpyAsync(hn.data(), dnodes.ptr, (size_t)m * 16, cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaMemcpyAsync(out_weights, dw.ptr, (size_t)m * 32, cudaMemcpyDeviceToHost, st));
    SG_CUDA(cudaMemcpyAsync(hs.data(), dstat.ptr, (size_t)m, cudaMemcpyDeviceToHost, st));
  }
  SG_CUDA(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < m * 4; ++i) out_nodes[i] = hn[i];
  if (out_status) std::copy(hs.begin(), hs.end(), out_status);
  for (int64_t i = 0; i < m; ++i)
    if (hs[i]) {
      if (out_first_bad) *out_first_bad = i;
      throw_error(SG_DOMAIN_ERROR, "NotLocated: target row %lld has a bilinear node outside the local mesh",
                  (long long)i);
    }
  if (out_stencil) {
    auto s = std::make_unique<Stencil>();
    s->device = device;
    s->m = m;
    s->k = 4;
    s->source_nnodes = n_nodes;
    stencil_finalize(s.get(), dnodes.as<int32_t>(), dw.as<double>(), st);
    *out_stencil = registry_put(s.release());
  }
  SG_API_END
}
