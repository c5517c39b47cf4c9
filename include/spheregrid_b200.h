/*
 * spheregrid_b200.h — flat C-ABI of the B200-native remap + halo-exchange hot path.
 *
 * This is the drop-in boundary for the `spheregrid` reference (Python, numpy/scipy,
 * /root/reference/pkg/src/spheregrid).  The reference has no native binding for the hot
 * path; its only binding layer is the TypeScript "FFI" in pkg/frontend, whose conventions
 * this header follows:
 *   - every call returns an int32 status: 0 ok, 1 domain error, 2 invalid handle,
 *     3 invalid argument                            (frontend/src/errors.ts:7-16,
 *                                                    SPEC.md capi StatusCode)
 *   - sg_last_error() copies the calling thread's last message (SPEC.md capi
 *     "Error text is copied into a caller-readable buffer per call context").  Domain
 *     errors are prefixed with the reference exception class name, e.g.
 *     "NotLocated: target point 17 not located ..." (errors.py:8-100), so a binding can
 *     re-raise the reference class.
 *   - opaque uint64 handles from a registry; never reused; double release -> status 2;
 *     sg_registry_count() is the leak probe                (frontend/src/registry.ts:15-35)
 *   - caller-owned host arrays cross as pointer + length and are copied on call; device
 *     buffers are owned by library handles.  No torch / numpy types in any signature.
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/pkg/src/spheregrid/).  Streams are cudaStream_t passed as uint64
 * (0 = the legacy default stream).
 */
#ifndef SPHEREGRID_B200_H
#define SPHEREGRID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_OK 0
#define SG_DOMAIN_ERROR 1
#define SG_INVALID_HANDLE 2
#define SG_INVALID_ARGUMENT 3

/* ---- runtime / registry (frontend/src/registry.ts:15-35, errors.ts:7-16) ---------------- */
int32_t sg_version(char* buf, size_t n);
int32_t sg_last_error(char* buf, size_t n);
int32_t sg_registry_count(int64_t* out_live);
int32_t sg_release(uint64_t handle);
int32_t sg_device_count(int32_t* out_count);
int32_t sg_device_uuid(int32_t device, uint8_t* out_uuid, size_t n);
int32_t sg_stream_synchronize(int32_t device, uint64_t stream);

/* ---- Field device mirror (field.py:77-162) ---------------------------------------------
 * Device storage of a (npts, levels) Field: one allocation, levels contiguous per point,
 * dense rows (pitch == levels: the reference host layout, field.py:161).  The pitch is
 * returned so callers never assume it.
 *   sg_field_alloc  <- Field.allocate_device        (field.py:99-105)
 *   sg_field_h2d    <- Field.update_device           (field.py:134-140)   host rows unpadded
 *   sg_field_d2h    <- Field.update_host             (field.py:126-132)
 *   sg_field_h2d_rows / sg_field_d2h_rows: the same for a contiguous row range.           */
int32_t sg_field_alloc(int32_t device, int64_t npts, int32_t levels, int32_t itemsize,
                       uint64_t* out_field, int64_t* out_pitch_elems, uint64_t* out_devptr);
int32_t sg_field_h2d(uint64_t field, const void* host, uint64_t stream);
int32_t sg_field_d2h(uint64_t field, void* host, uint64_t stream);
int32_t sg_field_h2d_rows(uint64_t field, int64_t row0, int64_t nrows, const void* host,
                          uint64_t stream);
int32_t sg_field_d2h_rows(uint64_t field, int64_t row0, int64_t nrows, void* host,
                          uint64_t stream);
/* runs: nruns (row0, nrows) pairs; copies host[row0 : row0+nrows] of the full (npts, levels)
 * host array into the same device rows (the host-field halo exchange uploads only the rows
 * its peers read, functionspace.py:107-118). */
int32_t sg_field_h2d_row_runs(uint64_t field, const int64_t* runs, int64_t nruns, const void* host,
                              uint64_t stream);
/* pinned, mapped host buffers (cudaHostAlloc) for asynchronous, full-rate h2d/d2h and the
 * GPU gather of sg_remap_execute_host; sg_host_alloc_flags: bit 0 write-combined, bit 1
 * zero-filled (the host mirrors create_field allocates, field.py:171).  CUDA events for
 * timing on the launching stream. */
int32_t sg_host_alloc(size_t bytes, uint64_t* out_ptr);
int32_t sg_host_alloc_flags(size_t bytes, int32_t flags, uint64_t* out_ptr);
int32_t sg_host_free(uint64_t ptr);
int32_t sg_host_register(uint64_t ptr, size_t bytes);
int32_t sg_host_unregister(uint64_t ptr);
int32_t sg_event_create(int32_t device, uint64_t* out_event);
int32_t sg_event_record(uint64_t event, uint64_t stream);
int32_t sg_event_elapsed_ms(uint64_t start, uint64_t end, float* out_ms);
/* streams (non-blocking; released with sg_release), cross-stream waits on events, and CUDA
 * graphs of a captured steady-state step (the multi-GPU exchange + apply). */
int32_t sg_stream_create(int32_t device, uint64_t* out_handle, uint64_t* out_stream);
int32_t sg_stream_wait_event(uint64_t stream, uint64_t event);
int32_t sg_enable_peer_access(int32_t device, int32_t peer);
int32_t sg_graph_begin(int32_t device, uint64_t stream);
int32_t sg_graph_end(int32_t device, uint64_t stream, uint64_t* out_graph);
int32_t sg_graph_launch(uint64_t graph, uint64_t stream);
int32_t sg_field_info(uint64_t field, int32_t* out_device, int64_t* out_npts,
                      int32_t* out_levels, int64_t* out_pitch_elems, uint64_t* out_devptr);

/* ---- stencil search + weights (interp.py:74-117 MeshLocator, interp.py:154-203) ---------
 * sg_locator_create <- MeshLocator.__init__ (interp.py:79-88): uploads node xyz (n,3) f64
 *   and the element CSR (mesh.py:310-319), splits quads at the lowest local index
 *   (mesh.py:395-403), and builds a latitude-band / longitude-bin search structure on the
 *   device (the B200 replacement for the cKDTree + incidence lists).
 * sg_locator_locate <- MeshLocator.locate (interp.py:102-117), batched: per point the
 *   element id, the local corner triple, or -1 (NotLocated), -2 (DegenerateTriangle: a
 *   degenerate triangle among the reference's kNN candidates, interp.py:34-43), -3 (more
 *   overlapping candidates than the exact emulation holds).  Winner = max over containing
 *   triangles (score = min of the three signed tests >= -CONTAIN_EPS) of the score; exact
 *   ties -> lowest local element id, then triangle index.  Meshes with
 *   degenerate triangles are decided per point as the k = 8 / min(32, n) nearest-node search
 *   would (node ranks by brute force; exact distance ties at the k-th place unpinned).
 * sg_remap_build <- build_remap (interp.py:154-203): locate + gnomonic barycentric weights
 *   (interp.py:61-71) + scale (interp.py:194) + optional nearest-node fallback
 *   (interp.py:179-190).  Returns a device stencil handle for sg_remap_apply and copies the
 *   InterpolationWeights arrays (interp.py:120-133) to the caller's host buffers.
 *   out_status[k]: 0 located, 1 not located (fallback row if allow_fallback),
 *   2 degenerate candidate triangle, 3 singular vertex matrix, 4 zero weight sum,
 *   5 undecidable (over 96 overlapping candidate triangles; SpheregridError).
 *   On status SG_DOMAIN_ERROR *out_first_bad is the first (ascending) offending row and
 *   the message carries the reference exception class (NotLocated / DegenerateTriangle).
 * sg_stencil_create: device stencil from host arrays (an InterpolationWeights built
 *   elsewhere, e.g. the reference's own build_remap output).                               */
int32_t sg_locator_create(int32_t device, const double* node_xyz, int64_t n_nodes,
                          const int64_t* elem_offsets, const int64_t* elem_indices,
                          int64_t n_elems, uint64_t* out_locator);
int32_t sg_locator_stats(uint64_t locator, int64_t* out_ntri, int64_t* out_nbins,
                         int64_t* out_nentries, double* out_band_rad);
int32_t sg_locator_locate(uint64_t locator, const double* points, int64_t m,
                          int64_t* out_elem, int64_t* out_corners);
int32_t sg_remap_build(uint64_t locator, const double* target_xyz, int64_t m,
                       int64_t source_nnodes, int32_t allow_fallback, uint64_t* out_stencil,
                       int64_t* out_nodes, double* out_weights, double* out_scale,
                       uint8_t* out_fallback, uint8_t* out_status, int64_t* out_first_bad);
int32_t sg_stencil_create(int32_t device, const int64_t* nodes, const double* weights,
                          int64_t m, int64_t source_nnodes, uint64_t* out_stencil);
/* k-point stencils: k = 3 (FE) or 4 (structured bilinear); nodes/weights are [m][k]. */
int32_t sg_stencil_create_k(int32_t device, const int64_t* nodes, const double* weights,
                            int64_t m, int32_t k, int64_t source_nnodes, uint64_t* out_stencil);
/* Structured-bilinear stencils (BASELINE configs[4]; no reference counterpart — defined in
 * csrc/bilinear.cu and restated in oracle/oracle.py:bilinear_stencil, parity unpinned vs
 * the reference): bracketing rows of the source grid, linear in longitude per row, linear
 * in latitude, polar caps through the pole nodes.  node_global: the local mesh's global ids
 * (mesh.py node_global) so the 4 nodes come back as local rows; target_lonlat (m, 2) in
 * degrees.  NotLocated (status 1, *out_first_bad) if a node is not in the local mesh. */
int32_t sg_bilinear_build(int32_t device, int32_t nrows, const double* lat_deg,
                          const int64_t* nlons, int32_t has_poles, const int64_t* node_global,
                          int64_t n_nodes, const double* target_lonlat, int64_t m,
                          uint64_t* out_stencil, int64_t* out_nodes, double* out_weights,
                          uint8_t* out_status, int64_t* out_first_bad);
int32_t sg_stencil_info(uint64_t stencil, int64_t* out_m, int64_t* out_source_nnodes,
                        int64_t* out_distinct_sources);

/* ---- apply (interp.py:206-228 apply_remap) ------------------------------------------------
 * dst[t, :] = (w0*src[n0, :] + w1*src[n1, :]) + w2*src[n2, :], every product and sum
 * rounded separately (bitwise equal to the numpy expression at interp.py:219-223), for
 * nfields source/target field pairs sharing the stencil.  ShapeMismatch (status 1) with
 * the reference messages when npts / levels disagree (interp.py:208-217).
 * variant: 0 = default (warp per target, vector loads), 2 = TMA bulk-copy (cp.async.bulk)
 * staged gather, producer warp + 16 consumer warps, 1 CTA/SM; 6 = the same with 8-target
 * tiles, 2 CTAs/SM; 3 = warp per target, 8-B loads; 4 / 5 = 8-B loads with L2::256B /
 * L2::128B prefetch-size hints.                                                            */
int32_t sg_remap_apply(uint64_t stencil, const uint64_t* src_fields,
                       const uint64_t* dst_fields, int32_t nfields, int32_t variant,
                       uint64_t stream);
/* The same for targets [t0, t1) only (pipelines, overlap of interior/boundary targets). */
int32_t sg_remap_apply_range(uint64_t stencil, const uint64_t* src_fields,
                             const uint64_t* dst_fields, int32_t nfields, int64_t t0,
                             int64_t t1, int32_t variant, uint64_t stream);
/* The same for an arbitrary target list (device int32 array of `count` target rows), e.g.
 * the interior / boundary targets of a partition. */
int32_t sg_remap_apply_list(uint64_t stencil, const uint64_t* src_fields,
                            const uint64_t* dst_fields, int32_t nfields,
                            const int32_t* dev_targets, int64_t count, int32_t variant,
                            uint64_t stream);
/* apply_remap with HOST buffers (the reference's call shape, interp.py:206-228): host
 * source rows -> device, apply, device -> host target rows, as an nchunks-deep pipeline
 * on three streams (h2d of source-row chunk c, apply of the targets whose stencils lie in
 * chunks <= c, d2h of those target rows).  Unreferenced gaps of < 64 rows are copied
 * through (*out_rows_copied).  host_src/host_dst: dense (npts, levels) C-order fp64, ideally
 * pinned (sg_host_alloc).  Synchronous: returns when host_dst holds the result. */
int32_t sg_remap_execute_host(uint64_t stencil, const uint64_t* src_fields,
                              const uint64_t* dst_fields, int32_t nfields,
                              const uint64_t* host_src, const uint64_t* host_dst,
                              int32_t nchunks, int32_t variant, int32_t flags,
                              int64_t* out_rows_copied);
/* flags bit 0 (compact): pack exactly the referenced source rows on the host (library thread
 * pool, pinned 3-slot staging ring) and apply from a compact device copy with a renumbered
 * stencil — PCIe carries U rows instead of every row (77 % at cfg3/cfg2).
 * flags bit 1 (zero-copy): the apply kernel reads source rows directly from the pinned host
 * array over PCIe and writes target rows directly into the pinned host array (mapped
 * pinned memory required, e.g. sg_host_alloc); no staging and no copy engines.
 * flags bit 2 (gather, the default for page-locked sources): a GPU kernel pulls exactly the
 * referenced source rows out of the pinned, mapped host array with cp.async.bulk copies into a
 * compact device copy (no host CPU work), pipelined with the apply and the d2h.
 * flags bit 3 (with bit 2): warp-per-row loads instead of bulk copies (comparison only).
 * flags bits 8-15 (compact): every n-th chunk copied whole by one DMA instead of packed. */

/* ---- halo exchange (functionspace.py:58-118) ---------------------------------------------
 * sg_halo_plan_create <- HaloExchangePlan (functionspace.py:47-55): per peer (ascending),
 *   the owned rows sent (owner-local, requester order, functionspace.py:82-93), the ghost
 *   rows received (local, (halo, gidx) order, functionspace.py:66-72) and, for the ghost
 *   rows, their index on the owner (mesh.py:303-308 node_remote).
 * sg_halo_pack   <- the send loop (functionspace.py:113-114): writes every peer's payload
 *   into one device buffer, peers ascending, each payload (n_send, L) C-order — byte-equal
 *   to f.host[send[peer]].tobytes().
 * sg_halo_unpack <- the receive loop (functionspace.py:115-117).
 * sg_halo_pull: fused pack + transfer + unpack over peer memory: ghost rows are read
 *   straight from each owner's device field (same device, NVLink P2P in one process, or a
 *   CUDA-IPC mapping) — one kernel, no staging.  peer_ptrs/peer_pitch indexed by plan peer.
 * sg_halo_exchange_nccl: pack -> grouped ncclSend/ncclRecv per peer -> unpack on one
 *   stream (NCCL loaded lazily with dlopen).                                                */
int32_t sg_halo_plan_create(int32_t device, int64_t nnodes, int32_t npeers,
                            const int32_t* peers, const int64_t* send_counts,
                            const int64_t* send_rows, const int64_t* recv_counts,
                            const int64_t* recv_rows, const int64_t* recv_remote_rows,
                            uint64_t* out_plan);
int32_t sg_halo_plan_info(uint64_t plan, int64_t* out_nsend, int64_t* out_nrecv);
int32_t sg_halo_pack(uint64_t plan, uint64_t field, void* dev_sendbuf, uint64_t stream);
int32_t sg_halo_unpack(uint64_t plan, uint64_t field, const void* dev_recvbuf,
                       uint64_t stream);
int32_t sg_halo_pull(uint64_t plan, uint64_t field, const uint64_t* peer_ptrs,
                     const int64_t* peer_pitch_elems, uint64_t stream);

/* Fused exchange + apply: applies targets [t0, t1) reading every ghost stencil row straight
 * from its owner's field (peer_ptrs/peer_pitch_elems by plan peer slot) — the halo exchange
 * of functionspace.py:107-118 and the apply of interp.py:206-228 in one kernel, no ghost
 * copy.  Caller guarantees the owners' rows are final (barrier) while it runs. */
int32_t sg_remap_apply_fused(uint64_t stencil, uint64_t plan, uint64_t src_field,
                             uint64_t dst_field, int64_t t0, int64_t t1,
                             const uint64_t* peer_ptrs, const int64_t* peer_pitch_elems,
                             uint64_t stream);
int32_t sg_remap_apply_fused_list(uint64_t stencil, uint64_t plan, uint64_t src_field,
                                  uint64_t dst_field, const int32_t* dev_targets, int64_t count,
                                  const uint64_t* peer_ptrs, const int64_t* peer_pitch_elems,
                                  uint64_t stream);
int32_t sg_nccl_unique_id(uint8_t* out_id, size_t n);
int32_t sg_comm_create(int32_t device, int32_t nranks, int32_t rank, const uint8_t* id,
                       size_t n, uint64_t* out_comm);
int32_t sg_halo_exchange_nccl(uint64_t plan, uint64_t field, uint64_t comm,
                              uint64_t stream);
/* Stream-ordered barrier (ncclAllReduce of one word on `stream`): fences the fused
 * exchange+apply's peer reads without a host round trip; graph-capturable. */
int32_t sg_comm_barrier(uint64_t comm, uint64_t stream);
/* one process, several GPUs (in-process ranks): ncclCommInitAll over devices[0..ndev), one
 * communicator handle per device in out_comms[rank] (SURVEY.md §8(b) sg_comm_init_all). */
int32_t sg_comm_init_all(int32_t ndev, const int32_t* devices, uint64_t* out_comms);
/* NCCL's own view of a communicator (ncclCommCount / ncclCommUserRank / ncclCommCuDevice) and
 * the loaded NCCL's version code; any out pointer may be NULL. */
int32_t sg_comm_info(uint64_t comm, int32_t* out_nranks, int32_t* out_rank, int32_t* out_device,
                     int32_t* out_version);

/* Fused distributed step with device-side signalling (csrc/step.cu): the halo exchange of
 * functionspace.py:107-118 and the apply of interp.py:206-228 for one rank as one kernel,
 * ordered like cli.py:138-144 (owners' rows final before ghosts are read) without host or
 * NCCL barriers.  Each rank owns a signal (2*nranks+4 uint64 words: ready[r], done[r], epoch,
 * current, count, error) that its peers write through NVLink P2P / CUDA-IPC pointers.
 *   sg_step_create: peer_* by plan peer slot (the owner's source field pointer + pitch, the
 *     peer's signal words); targets whose stencil reads a ghost row wait for their owners'
 *     ready word and read that row from the owner's field.
 *   sg_step_launch: one signal kernel + one step kernel over n steps of ONE device.  n = 1 and
 *     wait_done = 1 with one GPU per rank; n > 1 (every rank of a single-GPU emulation in one
 *     launch) requires wait_done = 0.
 *   sg_step_check: status 1 if a wait timed out (a peer never signalled); waits are bounded by
 *     sg_step_set_timeout (default 10 s). */
int32_t sg_signal_create(int32_t device, int32_t nranks, int32_t rank, uint64_t* out_signal);
int32_t sg_signal_ptr(uint64_t signal, uint64_t* out_dev_ptr);
int32_t sg_signal_ipc_handle(uint64_t signal, uint8_t* out_handle, size_t n);
int32_t sg_signal_read(uint64_t signal, uint64_t* out_words, int64_t n);
int32_t sg_signal_write(uint64_t signal, const uint64_t* words, int64_t n);  /* tests / measurement */
int32_t sg_step_create(uint64_t stencil, uint64_t plan, uint64_t src_field, uint64_t dst_field,
                       uint64_t signal, const uint64_t* peer_ptrs, const int64_t* peer_pitch_elems,
                       const uint64_t* peer_flag_ptrs, uint64_t* out_step);
int32_t sg_step_info(uint64_t step, int64_t* out_m, int64_t* out_n_boundary);
int32_t sg_step_launch(const uint64_t* steps, int32_t n, int32_t wait_done, uint64_t stream);
/* Test/emulation entry: the same launch over every rank of a single-GPU emulation WITH the tail
 * waits (wait_done = 1) as one cooperative launch — all blocks co-resident, so a rank's finisher
 * may spin on the done words of readers in the same grid.  Status 1 if the grid does not fit
 * the GPU at once (small problems only). */
int32_t sg_step_launch_cooperative(const uint64_t* steps, int32_t n, uint64_t stream);
int32_t sg_step_check(uint64_t step, uint64_t* out_error, uint64_t* out_epoch);
int32_t sg_step_set_timeout(uint64_t step, uint64_t timeout_ns);
/* The halo exchange alone, signalled (functionspace.py:107-118; cfg4): one signal kernel + one
 * pull kernel per rank — a warp per ghost row waits for its owner's ready word and copies the
 * owner's row (recv_remote) through the peer pointer; the last row publishes done.  Same
 * signal words, launch rules (n > 1 on one GPU => wait_done = 0) and timeout as the step;
 * sg_exchange_signal returns the signal handle (check its error word with sg_signal_read). */
int32_t sg_exchange_create(uint64_t plan, uint64_t field, uint64_t signal, const uint64_t* peer_ptrs,
                           const int64_t* peer_pitch_elems, const uint64_t* peer_flag_ptrs,
                           uint64_t* out_exchange);
int32_t sg_exchange_launch(const uint64_t* exchanges, int32_t n, int32_t wait_done, uint64_t stream);
int32_t sg_exchange_launch_cooperative(const uint64_t* exchanges, int32_t n, uint64_t stream);
int32_t sg_exchange_set_timeout(uint64_t exchange, uint64_t timeout_ns);
int32_t sg_exchange_signal(uint64_t exchange, uint64_t* out_signal);

/* Partition-invariant digest of owned rows [row0, row0+nrows) whose global ids are gids
 * (functionspace.py:233-254): the wrapping u64 sum of splitmix64(gid*G + (level+1)*Lv ^ bits);
 * the caller sums the partials over ranks (gather_to_root + broadcast, as the reference). */
int32_t sg_field_checksum(uint64_t field, int64_t row0, int64_t nrows, const int64_t* gids,
                          uint64_t* out_partial);

/* gather_field / scatter_field on the device (functionspace.py:185-224): indexed row copy
 *   dst[dst_idx ? dst_idx[i] : i] = src[src_idx ? src_idx[i] : i], i < n, rows of row_bytes
 * (a multiple of 4); indices are device int64 arrays (NULL = identity); src / dst may be peer
 * memory (P2P or CUDA IPC mappings). */
int32_t sg_rows_copy(int32_t device, uint64_t dst, int64_t dst_pitch_bytes, const int64_t* dst_idx_dev,
                     uint64_t src, int64_t src_pitch_bytes, const int64_t* src_idx_dev, int64_t n,
                     int64_t row_bytes, uint64_t stream);

/* CUDA IPC for the multi-process pull path (one process per GPU). */
int32_t sg_ipc_handle(uint64_t field, uint8_t* out_handle, size_t n);
int32_t sg_ipc_open(int32_t device, const uint8_t* handle, size_t n, uint64_t* out_ptr);
int32_t sg_ipc_close(int32_t device, uint64_t ptr);

/* ---- host-side setup, native -------------------------------------
 * sg_meshgen_create <- generate_mesh (mesh.py:229-338) minus coordinates: serial strip-merge
 *   topology (mesh.py:142-215), element halo levels + BFS (mesh.py:247-278), local node
 *   numbering (mesh.py:280-308) and local connectivity (mesh.py:310-319).  Results stay in
 *   the handle; sg_meshgen_fetch copies them out.
 * sg_matching_partition <- PointCloudIndex.query + matching_partition (partition.py:53-88):
 *   nearest master grid point with the 1e-12 relative tie window resolved to the smallest
 *   global index, using the master grid's row structure instead of a kd-tree.               */
int32_t sg_meshgen_create(int32_t nrows, const int64_t* nlons, int32_t include_pole,
                          const int32_t* part_of, int64_t npts, int32_t nparts, int32_t part,
                          int32_t halo, uint64_t* out_mesh, int64_t* out_nnodes,
                          int64_t* out_nowned, int64_t* out_nelems, int64_t* out_nindices);
int32_t sg_meshgen_fetch(uint64_t mesh, int64_t* node_global, int32_t* node_part,
                         int64_t* node_remote, uint8_t* node_ghost, int16_t* node_halo,
                         int64_t* elem_offsets, int64_t* elem_indices, int16_t* elem_halo,
                         int64_t* elem_serial_id);
int32_t sg_matching_partition(int32_t nrows, const double* master_lat_deg,
                              const int64_t* master_nlons, const double* master_xyz,
                              const double* target_xyz, int64_t m, int32_t nthreads,
                              int64_t* out_index);

#ifdef __cplusplus
}
#endif
#endif /* SPHEREGRID_B200_H */
