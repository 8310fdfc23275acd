// Multi-GPU slab exchange over peer memory ("fuse" option):
// each rank maps its y/z neighbours' grid buffers and flag words through
// CUDA IPC; after the boundary tile bands of step t are computed, the copy
// engine writes the slab's r outermost rows straight into the neighbours'
// halo rows (the buffer they read at step t+1) and a stream memory operation
// bumps the neighbour's flag.  The neighbour's compute stream waits on its own
// flag before step t+1.  Everything is stream-ordered: no NCCL, no host
// synchronisation, one host call per step.
//
// Hazards (slab boundaries are whole tile bands, band >= r):
//   RAW  step t+1 of rank k reads halo rows written by the neighbours' step-t
//        exchange -> cuStreamWaitValue32(flag >= t+1) before step t+1.
//   WAR  the neighbour's step-(t+1) exchange overwrites rank k's buf[t&1]
//        halo, read only by rank k's step-t BOUNDARY launch, which completed
//        before rank k signalled step t (the neighbour waited for that signal
//        before its step-t+1 boundary launch, which precedes its exchange).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "spider_internal.h"

namespace spd {

typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

struct DriverFns {
  WaitValueFn wait = nullptr;
  WriteValueFn write = nullptr;
  AddrRangeFn range = nullptr;
};

static const DriverFns& driver() {
  static DriverFns f;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f.wait = reinterpret_cast<WaitValueFn>(p);
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f.write = reinterpret_cast<WriteValueFn>(p);
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f.range = reinterpret_cast<AddrRangeFn>(p);
  });
  return f;
}

static int cu_err(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return SPD_OK;
  return set_error(SPD_ECUDA, "%s failed (CUresult %d)", what, (int)r);
}
static int rt_err(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SPD_OK;
  return set_error(SPD_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace spd

struct spd_slab {
  const spd_plan* plan;
  spd_grid_desc g;
  void* buf[2];
  int band;       // tile band height (rows 2D / planes 3D)
  int64_t extent; // local rows (2D) / planes (3D)
  int64_t unit;   // elements per stored row / plane
  int r;
  bool has_up, has_dn;
  void* up_buf[2];
  void* dn_buf[2];
  int64_t up_extent, dn_extent;
  unsigned int* up_flag;  // neighbour's flag word written by us (its "from down" / "from up")
  unsigned int* dn_flag;
  unsigned int* my_flags; // [0] from up, [1] from down (written by the neighbours)
  unsigned int wait_flags;
  cudaEvent_t boundary_done;
  // one launch per step (spd_step_edge_first): edge bands first, published
  // per band, then the interior forward (even steps) / backward (odd steps,
  // L2 reuse); the copy engine waits on the edge bands' counters instead of
  // a kernel boundary
  int n_bands, per_band;
  unsigned int* band_done = nullptr; // device: cumulative finished tiles per band
};

extern "C" {

int spd_ipc_export(const void* ptr, void* handle, int64_t* offset) {
  using namespace spd;
  if (!ptr || !handle || !offset) return set_error(SPD_EINVAL, "null argument");
  const DriverFns& f = driver();
  if (!f.range) return set_error(SPD_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  int rc = cu_err(f.range(&base, &size, (CUdeviceptr)ptr), "cuMemGetAddressRange");
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  rc = rt_err(cudaIpcGetMemHandle(&h, (void*)base), "cudaIpcGetMemHandle");
  if (rc) return rc;
  std::memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)((CUdeviceptr)ptr - base);
  return SPD_OK;
}

int spd_ipc_open(const void* handle, int64_t offset, void** ptr, void** base) {
  using namespace spd;
  if (!handle || !ptr || !base) return set_error(SPD_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* b = nullptr;
  int rc = rt_err(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  if (rc) return rc;
  *base = b;
  *ptr = (char*)b + offset;
  return SPD_OK;
}

int spd_ipc_close(void* base) {
  using namespace spd;
  return rt_err(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle");
}

int spd_slab_create(const spd_plan* plan, const spd_grid_desc* g, void* buf0, void* buf1, void* my_flags,
                    void* up_buf0, void* up_buf1, const spd_grid_desc* up_g, void* up_flags, void* dn_buf0,
                    void* dn_buf1, const spd_grid_desc* dn_g, void* dn_flags, spd_slab** out) {
  using namespace spd;
  if (!plan || !g || !buf0 || !buf1 || !my_flags || !out) return set_error(SPD_EINVAL, "null argument");
  if (g->dims == 1) return set_error(SPD_EINVAL, "1D grids have no slab halo");
  const DriverFns& f = driver();
  if (!f.wait || !f.write) return set_error(SPD_ECUDA, "stream memory operations unavailable");
  int32_t info[16];  // spd_plan_info writes 11 entries
  int rc = spd_plan_info(plan, info);
  if (rc) return rc;
  spd_slab* s = new spd_slab();
  s->plan = plan;
  s->g = *g;
  s->buf[0] = buf0;
  s->buf[1] = buf1;
  s->band = g->dims == 3 ? info[5] : info[6];
  s->extent = g->dims == 3 ? g->nz : g->ny;
  s->unit = g->dims == 3 ? g->plane : g->pitch;
  s->r = g->halo;
  s->my_flags = (unsigned int*)my_flags;
  s->has_up = up_buf0 != nullptr;
  s->has_dn = dn_buf0 != nullptr;
  if (s->has_up) {
    if (!up_g || up_g->pitch != g->pitch || up_g->origin != g->origin || (g->dims == 3 && up_g->plane != g->plane) ||
        !up_flags)
      return delete s, set_error(SPD_EINVAL, "up neighbour layout differs");
    s->up_buf[0] = up_buf0;
    s->up_buf[1] = up_buf1;
    s->up_extent = up_g->dims == 3 ? up_g->nz : up_g->ny;
    s->up_flag = (unsigned int*)up_flags + 1;  // its "from down" word
  }
  if (s->has_dn) {
    if (!dn_g || dn_g->pitch != g->pitch || dn_g->origin != g->origin || (g->dims == 3 && dn_g->plane != g->plane) ||
        !dn_flags)
      return delete s, set_error(SPD_EINVAL, "down neighbour layout differs");
    s->dn_buf[0] = dn_buf0;
    s->dn_buf[1] = dn_buf1;
    s->dn_extent = dn_g->dims == 3 ? dn_g->nz : dn_g->ny;
    s->dn_flag = (unsigned int*)dn_flags + 0;  // its "from up" word
  }
  if (s->extent < s->r || (s->has_dn && s->extent % s->band != 0))
    return delete s, set_error(SPD_EINVAL, "slab of %lld rows cannot exchange (band %d)", (long long)s->extent, s->band);
  // remote-write flush on the waits where the device supports it
  int dev = 0, can_flush = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&can_flush, cudaDevAttrCanFlushRemoteWrites, dev);
  s->wait_flags = CU_STREAM_WAIT_VALUE_GEQ | (can_flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
  rc = rt_err(cudaEventCreateWithFlags(&s->boundary_done, cudaEventDisableTiming), "event");
  if (rc) return delete s, rc;
  {
    const int tile_x = info[4] * info[0];  // n_tile * L (single-CTA geometry)
    const int64_t tiles_x = (g->nx + tile_x - 1) / tile_x;
    const int64_t tiles_y = g->dims == 3 ? (g->ny + info[6] - 1) / info[6] : 1;
    s->per_band = (int)(tiles_x * tiles_y);
    s->n_bands = (int)((s->extent + s->band - 1) / s->band);
    rc = rt_err(cudaMalloc(&s->band_done, sizeof(unsigned int) * s->n_bands), "counter alloc");
    if (!rc) rc = rt_err(cudaMemset(s->band_done, 0, sizeof(unsigned int) * s->n_bands), "counter reset");
    if (rc) return spd_slab_destroy(s), rc;
  }
  *out = s;
  return SPD_OK;
}

int spd_slab_destroy(spd_slab* s) {
  if (!s) return SPD_OK;
  cudaEventDestroy(s->boundary_done);
  if (s->band_done) cudaFree(s->band_done);
  delete s;
  return SPD_OK;
}

// Element offset of stored row / plane i (interior index; negative = halo).
static int64_t unit_start(const spd_grid_desc* g, int64_t unit, int64_t i) {
  return g->origin - (g->origin % unit) + i * unit;
}

int spd_slab_step(spd_slab* s, int t, void* compute_stream, void* comm_stream) {
  using namespace spd;
  if (!s) return set_error(SPD_EINVAL, "null slab");
  const DriverFns& f = driver();
  cudaStream_t cs = (cudaStream_t)compute_stream, xs = (cudaStream_t)comm_stream;
  const void* in = s->buf[t & 1];
  void* out = s->buf[(t + 1) & 1];
  // 1. this step reads halo rows the neighbours wrote in their step t-1
  if (t > 0) {
    if (s->has_up) {
      int rc = cu_err(f.wait((CUstream)cs, (CUdeviceptr)(s->my_flags + 0), (cuuint32_t)t, s->wait_flags), "wait up");
      if (rc) return rc;
    }
    if (s->has_dn) {
      int rc = cu_err(f.wait((CUstream)cs, (CUdeviceptr)(s->my_flags + 1), (cuuint32_t)t, s->wait_flags), "wait down");
      if (rc) return rc;
    }
  }
  // 2a. one launch, edge bands first and published per band; the copy engine
  //     starts on the edge rows while the interior is still being computed
  // Launch form (tools/ordered_time.py, cooled and interleaved, 1 B200; step
  // time vs a plain step): one edge-first launch publishing its edge tiles
  // costs B9 +4.9 %, W +4.7 %, B27 +25 % (system-scope publishing of 512
  // edge tiles); an edge launch + an interior launch costs B9 +8.3 %, W
  // +3.1 %, B27 +3.8 %.  So: two launches for 3D and for large slabs, one
  // launch for small 2D slabs.  SPD_SLAB_TWO_LAUNCH=0/1 overrides.
  const char* two_env = getenv("SPD_SLAB_TWO_LAUNCH");  // read per step: tests switch it in-process
  const bool two_launch = two_env ? atoi(two_env) != 0
                                  : (s->g.dims == 3 || (int64_t)s->per_band * s->n_bands >= 10000);
  // Fused peer stores: the edge tiles' epilogue writes the r outermost rows
  // straight into the neighbours' halo rows (NVLink stores; same layout), so
  // the comm stream only signals -- no copy.  Geometries without them (the
  // generic radii) keep the copy-engine exchange.  SPD_SLAB_COPY=1 forces it.
  const char* copy_env = getenv("SPD_SLAB_COPY");
  const bool fused = plan_peer_stores(s->plan) && !(copy_env && atoi(copy_env) != 0);
  PeerStores ps;
  ps.out[0] = s->has_up ? s->up_buf[(t + 1) & 1] : nullptr;
  ps.out[1] = s->has_dn ? s->dn_buf[(t + 1) & 1] : nullptr;
  ps.row[0] = s->up_extent;  // my row u -> the up neighbour's row up_extent + u (its bottom halo)
  ps.row[1] = -s->extent;    // my row u -> the down neighbour's row u - extent (its top halo)
  ps.rows = s->r;
  if ((s->has_up || s->has_dn) && !two_launch) {
    int rc0 = step_edge_first_ex(s->plan, &s->g, in, out, t & 1, s->band_done, 1, fused ? &ps : nullptr, cs);
    if (rc0) return rc0;
    const cuuint32_t target = (cuuint32_t)((int64_t)(t + 1) * s->per_band);
    const size_t bytes = (size_t)s->r * s->unit * 2;
    const uint16_t* o = (const uint16_t*)out;
    if (s->has_up) {
      int rc = cu_err(f.wait((CUstream)xs, (CUdeviceptr)(s->band_done + 0), target, CU_STREAM_WAIT_VALUE_GEQ),
                      "wait top band");
      if (rc) return rc;
      uint16_t* dst = (uint16_t*)s->up_buf[(t + 1) & 1] + unit_start(&s->g, s->unit, s->up_extent);
      if (!fused)
        rc = rt_err(cudaMemcpyAsync(dst, o + unit_start(&s->g, s->unit, 0), bytes, cudaMemcpyDeviceToDevice, xs),
                    "peer copy up");
      if (rc) return rc;
      rc = cu_err(f.write((CUstream)xs, (CUdeviceptr)s->up_flag, (cuuint32_t)(t + 1), CU_STREAM_WRITE_VALUE_DEFAULT),
                  "signal up");
      if (rc) return rc;
    }
    if (s->has_dn) {
      int rc = cu_err(f.wait((CUstream)xs, (CUdeviceptr)(s->band_done + s->n_bands - 1), target, CU_STREAM_WAIT_VALUE_GEQ),
                      "wait bottom band");
      if (rc) return rc;
      uint16_t* dst = (uint16_t*)s->dn_buf[(t + 1) & 1] + unit_start(&s->g, s->unit, -s->r);
      if (!fused)
        rc = rt_err(cudaMemcpyAsync(dst, o + unit_start(&s->g, s->unit, s->extent - s->r), bytes,
                                    cudaMemcpyDeviceToDevice, xs),
                    "peer copy down");
      if (rc) return rc;
      rc = cu_err(f.write((CUstream)xs, (CUdeviceptr)s->dn_flag, (cuuint32_t)(t + 1), CU_STREAM_WRITE_VALUE_DEFAULT),
                  "signal down");
      if (rc) return rc;
    }
    return SPD_OK;
  }
  // 2b. boundary bands (one launch), then the exchange on the comm stream
  const int64_t last = ((s->extent - 1) / s->band) * s->band;
  const bool split = last > s->band;
  int rc = split ? step_edges_ex(s->plan, &s->g, in, out, fused ? &ps : nullptr, cs)
                 : (fused ? step_edge_first_ex(s->plan, &s->g, in, out, t & 1, nullptr, 0, &ps, cs)
                          : spd_step_range(s->plan, &s->g, in, out, 0, s->extent, cs));
  if (rc) return rc;
  if (s->has_up || s->has_dn) {
    rc = rt_err(cudaEventRecord(s->boundary_done, cs), "event record");
    if (rc) return rc;
    rc = rt_err(cudaStreamWaitEvent(xs, s->boundary_done, 0), "stream wait event");
    if (rc) return rc;
    const size_t bytes = (size_t)s->r * s->unit * 2;
    const uint16_t* o = (const uint16_t*)out;
    if (s->has_up) {  // my first r rows -> up neighbour's bottom halo (rows extent_up ..)
      uint16_t* dst = (uint16_t*)s->up_buf[(t + 1) & 1] + unit_start(&s->g, s->unit, s->up_extent);
      if (!fused)
        rc = rt_err(cudaMemcpyAsync(dst, o + unit_start(&s->g, s->unit, 0), bytes, cudaMemcpyDeviceToDevice, xs),
                    "peer copy up");
      if (rc) return rc;
      rc = cu_err(f.write((CUstream)xs, (CUdeviceptr)s->up_flag, (cuuint32_t)(t + 1), CU_STREAM_WRITE_VALUE_DEFAULT),
                  "signal up");
      if (rc) return rc;
    }
    if (s->has_dn) {  // my last r rows -> down neighbour's top halo (rows -r ..)
      uint16_t* dst = (uint16_t*)s->dn_buf[(t + 1) & 1] + unit_start(&s->g, s->unit, -s->r);
      if (!fused)
        rc = rt_err(cudaMemcpyAsync(dst, o + unit_start(&s->g, s->unit, s->extent - s->r), bytes,
                                    cudaMemcpyDeviceToDevice, xs),
                    "peer copy down");
      if (rc) return rc;
      rc = cu_err(f.write((CUstream)xs, (CUdeviceptr)s->dn_flag, (cuuint32_t)(t + 1), CU_STREAM_WRITE_VALUE_DEFAULT),
                  "signal down");
      if (rc) return rc;
    }
  }
  // 3. interior bands overlap the exchange
  if (split) {
    rc = spd_step_range(s->plan, &s->g, in, out, s->band, last, cs);
    if (rc) return rc;
  }
  return SPD_OK;
}

// All steps of a run in one call (the host loop of one device; a process
// driving several devices runs one such call per device on its own thread).
int spd_slab_run(spd_slab* s, int t0, int steps, void* compute_stream, void* comm_stream) {
  using namespace spd;
  if (!s) return set_error(SPD_EINVAL, "null slab");
  if (t0 < 0 || steps < 1) return set_error(SPD_EINVAL, "bad step range (t0 %d, steps %d)", t0, steps);
  for (int t = t0; t < t0 + steps; ++t) {
    int rc = spd_slab_step(s, t, compute_stream, comm_stream);
    if (rc) return rc;
  }
  return SPD_OK;
}

// Direct peer access from `device` to `peer` (single-process multi-device
// slabs: the neighbours' buffers and flag words are plain device pointers).
int spd_peer_enable(int device, int peer) {
  using namespace spd;
  if (device == peer) return SPD_OK;
  int can = 0;
  int rc = rt_err(cudaDeviceCanAccessPeer(&can, device, peer), "cudaDeviceCanAccessPeer");
  if (rc) return rc;
  if (!can) return set_error(SPD_EUNSUPPORTED, "device %d cannot access peer device %d", device, peer);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the (non-sticky) error it recorded
    e = cudaSuccess;
  }
  cudaSetDevice(prev);
  return rt_err(e, "cudaDeviceEnablePeerAccess");
}

}  // extern "C"
