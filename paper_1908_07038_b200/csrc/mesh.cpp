// Native per-partition mesh topology: generate_mesh (mesh.py:229-338) without the
// coordinates (those stay in numpy on the host so their bits match the reference).
//
// Integer-only, bit-exact by construction:
//   serial topology       strip merge of adjacent rows + polar fans      mesh.py:142-215
//   ownership             blocks part_of, poles owned by the owners of gid 0 / npts-1
//                                                                         mesh.py:221-226
//   element halo levels   0 all owned, 1 some owned (halo >= 1), k = touches a node of a
//                         level < k element (BFS, one sweep per depth)    mesh.py:247-278
//   kept elements         ascending level, serial order within a level    mesh.py:280-282
//   local nodes           owned in global order ++ ghosts by (level, gid) mesh.py:284-298
//   node_remote           position of the gid in its owner's owned list    mesh.py:300-308
//   connectivity          CSR of local indices                            mesh.py:310-319
// The serial topology is cached per (row counts, poles) like _TOPO_CACHE (mesh.py:130).
#include <algorithm>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "host_pool.h"
#include "sg_internal.h"

namespace sg {
namespace {

struct Topology {
  int64_t nnodes = 0;  // npts (+2)
  std::vector<int64_t> off;   // nelem + 1
  std::vector<int32_t> nodes; // global ids
};

void merge_strip(int64_t o1, int64_t n1, int64_t o2, int64_t n2, Topology& t) {
  int64_t i1 = 0, i2 = 0;
  auto push = [&](std::initializer_list<int64_t> e) {
    for (int64_t g : e) t.nodes.push_back((int32_t)g);
    t.off.push_back((int64_t)t.nodes.size());
  };
  while (i1 < n1 || i2 < n2) {
    const bool can_n = i1 < n1, can_s = i2 < n2;
    bool adv_n;
    if (can_n && can_s) {
      const int64_t lhs = (i1 + 1) * n2, rhs = (i2 + 1) * n1;
      if (lhs == rhs) {
        push({o2 + i2, o2 + (i2 + 1) % n2, o1 + (i1 + 1) % n1, o1 + i1});
        ++i1;
        ++i2;
        continue;
      }
      adv_n = lhs < rhs;
    } else {
      adv_n = can_n;
    }
    if (adv_n) {
      push({o2 + i2 % n2, o1 + (i1 + 1) % n1, o1 + i1});
      ++i1;
    } else {
      push({o2 + i2, o2 + (i2 + 1) % n2, o1 + i1 % n1});
      ++i2;
    }
  }
}

std::mutex g_topo_mu;
std::map<std::pair<std::vector<int64_t>, int>, std::shared_ptr<Topology>> g_topo;

std::shared_ptr<Topology> serial_topology(const std::vector<int64_t>& nlons, bool poles) {
  std::lock_guard<std::mutex> lk(g_topo_mu);
  auto key = std::make_pair(nlons, poles ? 1 : 0);
  auto it = g_topo.find(key);
  if (it != g_topo.end()) return it->second;
  auto t = std::make_shared<Topology>();
  const int64_t nrows = (int64_t)nlons.size();
  std::vector<int64_t> roff(nrows + 1, 0);
  for (int64_t j = 0; j < nrows; ++j) roff[j + 1] = roff[j] + nlons[j];
  const int64_t npts = roff[nrows];
  t->nnodes = npts + (poles ? 2 : 0);
  t->off.push_back(0);
  size_t est = 0;
  for (int64_t j = 0; j + 1 < nrows; ++j) est += (size_t)(nlons[j] + nlons[j + 1]) * 4;
  t->nodes.reserve(est + (poles ? (size_t)(nlons.front() + nlons.back()) * 3 : 0));
  const int64_t np_ = npts, sp = npts + 1;
  if (poles) {
    const int64_t o0 = roff[0], n0 = nlons[0];
    for (int64_t i = 0; i < n0; ++i) {
      t->nodes.push_back((int32_t)(o0 + i));
      t->nodes.push_back((int32_t)(o0 + (i + 1) % n0));
      t->nodes.push_back((int32_t)np_);
      t->off.push_back((int64_t)t->nodes.size());
    }
  }
  for (int64_t j = 0; j + 1 < nrows; ++j) merge_strip(roff[j], nlons[j], roff[j + 1], nlons[j + 1], *t);
  if (poles) {
    const int64_t oL = roff[nrows - 1], nL = nlons[nrows - 1];
    for (int64_t i = 0; i < nL; ++i) {
      t->nodes.push_back((int32_t)(oL + (i + 1) % nL));
      t->nodes.push_back((int32_t)(oL + i));
      t->nodes.push_back((int32_t)sp);
      t->off.push_back((int64_t)t->nodes.size());
    }
  }
  g_topo.emplace(key, t);
  return t;
}

// Element and node passes run in blocks on a host thread pool (results are independent of the
// block split: every pass writes per-element slots, or sets node flags to one value per pass).
HostPool& mesh_pool() {
  static HostPool pool((int)std::max(1u, std::min(16u, std::thread::hardware_concurrency())) - 1);
  return pool;
}

template <class F>
void pfor(int64_t n, F&& body) {  // body(lo, hi) over [0, n) in blocks
  if (n <= 0) return;
  HostPool& pool = mesh_pool();
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(pool.size() * 4, (n + 32767) / 32768));
  if (nb == 1) {
    body((int64_t)0, n);
    return;
  }
  pool.parallel_for(nb, [&](int b) { body(n * b / nb, n * (b + 1) / nb); });
}

template <class T>
inline void set_relaxed(T* p, T v) {
  __atomic_store_n(p, v, __ATOMIC_RELAXED);
}
template <class T>
inline T get_relaxed(const T* p) {
  return __atomic_load_n(p, __ATOMIC_RELAXED);
}

struct MeshGen : Object {
  MeshGen() : Object(ObjKind::MeshGen) {}
  std::vector<int64_t> node_global, node_remote, elem_off, elem_idx, elem_serial;
  std::vector<int32_t> node_part;
  std::vector<uint8_t> node_ghost;
  std::vector<int16_t> node_halo, elem_halo;
  int64_t nowned = 0;
};

}  // namespace
}  // namespace sg

using namespace sg;

extern "C" {

int32_t sg_meshgen_create(int32_t nrows, const int64_t* nlons, int32_t include_pole, const int32_t* part_of,
                          int64_t npts, int32_t nparts, int32_t part, int32_t halo, uint64_t* out_mesh,
                          int64_t* out_nnodes, int64_t* out_nowned, int64_t* out_nelems, int64_t* out_nindices) {
  SG_API_BEGIN
  SG_REQUIRE(out_mesh && nlons && part_of, "null arguments");
  SG_REQUIRE(nrows >= 1, "need at least one row");
  SG_REQUIRE(nparts >= 1 && part >= 0 && part < nparts, "partition %d not in [0, %d)", part, nparts);
  SG_REQUIRE(halo >= 0, "negative halo");
  std::vector<int64_t> nl(nlons, nlons + nrows);
  int64_t sum = 0;
  for (int64_t n : nl) {
    SG_REQUIRE(n >= 1, "every row needs nlon >= 1");
    sum += n;
  }
  if (sum != npts)
    throw_error(SG_DOMAIN_ERROR, "InvalidDistribution: distribution sized %lld for a grid of %lld points",
                (long long)npts, (long long)sum);
  SG_REQUIRE(sum + 2 < INT32_MAX, "grid too large");
  auto topo = serial_topology(nl, include_pole != 0);
  const int64_t nn = topo->nnodes;
  const int64_t nelem = (int64_t)topo->off.size() - 1;
  // owners (mesh.py:221-226)
  std::vector<int32_t> owner(nn);
  for (int64_t g = 0; g < npts; ++g) {
    SG_REQUIRE(part_of[g] >= 0 && part_of[g] < nparts, "part_of[%lld] out of range", (long long)g);
    owner[g] = part_of[g];
  }
  if (include_pole) {
    owner[npts] = owner[0];
    owner[npts + 1] = owner[npts - 1];
  }
  std::vector<uint8_t> owned(nn);
  pfor(nn, [&](int64_t lo, int64_t hi) {
    for (int64_t g = lo; g < hi; ++g) owned[g] = owner[g] == part;
  });
  // element levels 0/1
  std::vector<int16_t> level(nelem, -1);
  const int64_t* off = topo->off.data();
  const int32_t* en = topo->nodes.data();
  pfor(nelem, [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      int64_t c = 0, k = off[e + 1] - off[e];
      for (int64_t i = off[e]; i < off[e + 1]; ++i) c += owned[en[i]];
      if (c == k) level[e] = 0;
      else if (c > 0 && halo >= 1) level[e] = 1;
    }
  });
  // nodes of kept elements: present; ghosts remember the first level that brings them in
  // (every writer of a pass stores the same value, so the block split does not matter)
  std::vector<uint8_t> present(nn, 0);
  std::vector<int16_t> intro(nn, 99);
  pfor(nelem, [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      if (level[e] < 0) continue;
      for (int64_t i = off[e]; i < off[e + 1]; ++i) {
        const int32_t g = en[i];
        set_relaxed(&present[g], (uint8_t)1);
        if (!owned[g]) set_relaxed(&intro[g], (int16_t)1);  // max(level, 1) == 1 here
      }
    }
  });
  std::vector<uint8_t> fresh(nelem, 0);
  for (int32_t depth = 2; depth <= halo; ++depth) {
    pfor(nelem, [&](int64_t lo, int64_t hi) {  // elements touching a present node
      for (int64_t e = lo; e < hi; ++e) {
        fresh[e] = 0;
        if (level[e] >= 0) continue;
        for (int64_t i = off[e]; i < off[e + 1]; ++i)
          if (present[en[i]]) {
            fresh[e] = 1;
            break;
          }
      }
    });
    pfor(nelem, [&](int64_t lo, int64_t hi) {
      for (int64_t e = lo; e < hi; ++e) {
        if (!fresh[e]) continue;
        level[e] = (int16_t)depth;
        for (int64_t i = off[e]; i < off[e + 1]; ++i) {
          const int32_t g = en[i];
          set_relaxed(&present[g], (uint8_t)1);
          if (!owned[g] && get_relaxed(&intro[g]) > depth) set_relaxed(&intro[g], (int16_t)depth);
        }
      }
    });
  }
  // kept elements: ascending level, serial order within a level (counting sort, stable)
  int16_t maxlv = 0;
  for (int64_t e = 0; e < nelem; ++e) maxlv = std::max(maxlv, level[e]);
  auto M = std::make_unique<MeshGen>();
  {
    std::vector<int64_t> cnt((size_t)maxlv + 2, 0);
    for (int64_t e = 0; e < nelem; ++e)
      if (level[e] >= 0) ++cnt[(size_t)level[e] + 1];
    for (size_t l = 1; l < cnt.size(); ++l) cnt[l] += cnt[l - 1];
    M->elem_serial.resize((size_t)cnt.back());
    for (int64_t e = 0; e < nelem; ++e)
      if (level[e] >= 0) M->elem_serial[(size_t)cnt[(size_t)level[e]]++] = e;
  }
  // local nodes
  for (int64_t g = 0; g < nn; ++g)
    if (owned[g]) M->node_global.push_back(g);
  M->nowned = (int64_t)M->node_global.size();
  std::vector<std::pair<int16_t, int64_t>> ghosts;
  for (int64_t g = 0; g < nn; ++g)
    if (!owned[g] && intro[g] != 99) ghosts.emplace_back(intro[g], g);
  std::sort(ghosts.begin(), ghosts.end());
  for (auto& gh : ghosts) M->node_global.push_back(gh.second);
  const int64_t nloc = (int64_t)M->node_global.size();
  std::vector<int32_t> local_of(nn, -1);
  for (int64_t i = 0; i < nloc; ++i) local_of[M->node_global[i]] = (int32_t)i;
  // position of every gid within its owner's owned list (count(owner[:g] == p))
  std::vector<int64_t> rank_in_part(nn), counter(nparts, 0);
  for (int64_t g = 0; g < nn; ++g) rank_in_part[g] = counter[owner[g]]++;
  M->node_part.resize(nloc);
  M->node_ghost.resize(nloc);
  M->node_halo.resize(nloc);
  M->node_remote.resize(nloc);
  for (int64_t i = 0; i < nloc; ++i) {
    const int64_t g = M->node_global[i];
    M->node_part[i] = owner[g];
    const bool gh = i >= M->nowned;
    M->node_ghost[i] = gh;
    M->node_halo[i] = gh ? ghosts[i - M->nowned].first : 0;
    M->node_remote[i] = gh ? rank_in_part[g] : i;
  }
  // local connectivity (CSR): offsets by prefix sum, indices filled in blocks
  const int64_t nkept = (int64_t)M->elem_serial.size();
  M->elem_off.resize((size_t)nkept + 1);
  M->elem_halo.resize((size_t)nkept);
  M->elem_off[0] = 0;
  for (int64_t k = 0; k < nkept; ++k) {
    const int64_t e = M->elem_serial[(size_t)k];
    M->elem_off[(size_t)k + 1] = M->elem_off[(size_t)k] + (off[e + 1] - off[e]);
    M->elem_halo[(size_t)k] = level[e];
  }
  M->elem_idx.resize((size_t)M->elem_off[(size_t)nkept]);
  pfor(nkept, [&](int64_t lo, int64_t hi) {
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t e = M->elem_serial[(size_t)k];
      int64_t o = M->elem_off[(size_t)k];
      for (int64_t i = off[e]; i < off[e + 1]; ++i) M->elem_idx[(size_t)o++] = local_of[en[i]];
    }
  });
  if (out_nnodes) *out_nnodes = nloc;
  if (out_nowned) *out_nowned = M->nowned;
  if (out_nelems) *out_nelems = (int64_t)M->elem_serial.size();
  if (out_nindices) *out_nindices = (int64_t)M->elem_idx.size();
  *out_mesh = registry_put(M.release());
  SG_API_END
}

int32_t sg_meshgen_fetch(uint64_t mesh, int64_t* node_global, int32_t* node_part, int64_t* node_remote,
                         uint8_t* node_ghost, int16_t* node_halo, int64_t* elem_offsets, int64_t* elem_indices,
                         int16_t* elem_halo, int64_t* elem_serial_id) {
  SG_API_BEGIN
  MeshGen* M = get<MeshGen>(mesh, ObjKind::MeshGen);
  auto cp = [](auto* dst, const auto& v) {
    if (dst) std::copy(v.begin(), v.end(), dst);
  };
  cp(node_global, M->node_global);
  cp(node_part, M->node_part);
  cp(node_remote, M->node_remote);
  cp(node_ghost, M->node_ghost);
  cp(node_halo, M->node_halo);
  cp(elem_offsets, M->elem_off);
  cp(elem_indices, M->elem_idx);
  cp(elem_halo, M->elem_halo);
  cp(elem_serial_id, M->elem_serial);
  SG_API_END
}

}  // extern "C"
