// Streams, cross-stream events and CUDA graphs for the multi-GPU step:
// the halo exchange runs on its own stream while the interior targets are applied, and the
// steady-state step (pack -> NCCL -> unpack | interior apply -> boundary apply) is captured
// once and replayed as one graph launch.
#include "cuda_util.cuh"

using namespace sg;

cudaEvent_t sg_event_raw(uint64_t h);  // field.cu

namespace {
struct Stream : Object {
  Stream() : Object(ObjKind::Stream) {}
  int device = 0;
  cudaStream_t s = nullptr;
  ~Stream() override {
    if (s) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (cur != device) cudaSetDevice(device);
      cudaStreamDestroy(s);
      if (cur != device && cur >= 0) cudaSetDevice(cur);
    }
  }
};
struct Graph : Object {
  Graph() : Object(ObjKind::Graph) {}
  int device = 0;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  ~Graph() override {
    if (exec) cudaGraphExecDestroy(exec);
    if (g) cudaGraphDestroy(g);
  }
};
}  // namespace

extern "C" {

int32_t sg_stream_create(int32_t device, uint64_t* out_handle, uint64_t* out_stream) {
  SG_API_BEGIN
  SG_REQUIRE(out_handle && out_stream, "null out pointer");
  DeviceScope ds(device);
  auto s = std::make_unique<Stream>();
  s->device = device;
  SG_CUDA(cudaStreamCreateWithFlags(&s->s, cudaStreamNonBlocking));
  *out_stream = reinterpret_cast<uint64_t>(s->s);
  *out_handle = registry_put(s.release());
  SG_API_END
}

int32_t sg_stream_wait_event(uint64_t stream, uint64_t event_handle) {
  SG_API_BEGIN
  SG_CUDA(cudaStreamWaitEvent(as_stream(stream), sg_event_raw(event_handle), 0));
  SG_API_END
}

// Let kernels on `device` dereference memory of `peer` (NVLink P2P within one process:
// run_ranks with one thread per GPU).  Idempotent.
int32_t sg_enable_peer_access(int32_t device, int32_t peer) {
  SG_API_BEGIN
  if (device == peer) return SG_OK;
  DeviceScope ds(device);
  int can = 0;
  SG_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) throw_error(SG_DOMAIN_ERROR, "CudaError: device %d cannot access device %d", device, peer);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  SG_CUDA(e);
  SG_API_END
}

int32_t sg_graph_begin(int32_t device, uint64_t stream) {
  SG_API_BEGIN
  DeviceScope ds(device);
  SG_CUDA(cudaStreamBeginCapture(as_stream(stream), cudaStreamCaptureModeThreadLocal));
  SG_API_END
}

int32_t sg_graph_end(int32_t device, uint64_t stream, uint64_t* out_graph) {
  SG_API_BEGIN
  SG_REQUIRE(out_graph, "null out pointer");
  DeviceScope ds(device);
  auto g = std::make_unique<Graph>();
  g->device = device;
  SG_CUDA(cudaStreamEndCapture(as_stream(stream), &g->g));
  SG_CUDA(cudaGraphInstantiate(&g->exec, g->g, 0));
  *out_graph = registry_put(g.release());
  SG_API_END
}

int32_t sg_graph_launch(uint64_t graph, uint64_t stream) {
  SG_API_BEGIN
  Graph* g = get<Graph>(graph, ObjKind::Graph);
  DeviceScope ds(g->device);
  SG_CUDA(cudaGraphLaunch(g->exec, as_stream(stream)));
  SG_API_END
}

}  // extern "C"
