// Device halo-exchange plan (functionspace.py:47-55), shared by halo.cu (exchange kernels)
// and fused.cu (apply that reads ghost rows straight from their owners).
#pragma once
#include <vector>

#include "cuda_util.cuh"

namespace sg {

constexpr int kMaxPeers = 64;

struct Plan : Object {
  Plan() : Object(ObjKind::Plan) {}
  int device = 0;
  int64_t nnodes = 0;
  std::vector<int32_t> peers;
  std::vector<int64_t> send_off, recv_off;   // per peer, npeers+1
  DevBuf send_rows, recv_rows, recv_remote;  // int32
  DevBuf recv_peer;                          // int32 plan-peer slot of every ghost row
  DevBuf sendbuf, recvbuf;                   // NCCL staging (lazily sized)
  // dense map of local rows [ghost_lo, nnodes): owner slot / owner row (-1: not a ghost)
  int64_t ghost_lo = 0;
  // every ghost's owner row is known (recv_remote given and >= 0): the pull and fused
  // kernels read owners' rows through it and are refused without it
  bool has_remote = false;
  DevBuf ghost_slot, ghost_row;              // int32
};

}  // namespace sg
