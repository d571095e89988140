// sgh_host.cu -- end-to-end batched transform on HOST buffers.
//
// The combination grids live in host memory (the iterated combination
// technique's solver owns them); they are streamed through the device in
// chunks: copy-in on one internal stream, the grouped transform on the
// caller's stream, copy-out on another, so PCIe traffic in both directions
// overlaps the transform of neighbouring chunks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/sgh.h"
#include "sgh_common.cuh"
#include "sgh_plan.hpp"

namespace sgh {

// transfer chunk (SGH_E2E_CHUNK_MB overrides, experiments)
static size_t chunk_bytes() {
  static size_t b = 0;
  if (!b) {
    const char *e = tuning_env("SGH_E2E_CHUNK_MB");
    const long mb = e ? atol(e) : 64;   // measured on C5: 64 MB 5.36, 128 MB 5.23, 512 MB 5.14, 2 GB 4.63 Gpoints/s
    b = size_t(mb >= 16 && mb <= 8192 ? mb : 64) << 20;
  }
  return b;
}

struct HostLayout {
  std::vector<size_t> grid_off;              // byte offset of each grid in the device buffer
  std::vector<std::pair<int64_t, int64_t>> chunks;  // [g0, g1)
  std::vector<size_t> table_off;             // byte offset of each chunk's task table
  size_t total = 0;
};

static sgh_status host_layout(const int32_t *levels, int32_t d, int64_t num_grids, uint32_t flags, HostLayout &L) {
  L.grid_off.resize(num_grids);
  size_t off = 0;
  size_t acc = 0;
  int64_t g0 = 0;
  for (int64_t g = 0; g < num_grids; ++g) {
    int64_t N = 0;
    sgh_status st = validate_levels(levels + g * d, d, &N);
    if (st != SGH_OK) return st;
    L.grid_off[g] = off;
    const size_t bytes = size_t(N) * 8;
    off += (bytes + 255) / 256 * 256;
    acc += bytes;
    if (acc >= chunk_bytes() || g == num_grids - 1) {
      L.chunks.push_back({g0, g + 1});
      g0 = g + 1;
      acc = 0;
    }
  }
  for (auto &c : L.chunks) {
    L.table_off.push_back(off);
    const size_t tb = batched_table_bytes(nullptr, levels + c.first * d, d, c.second - c.first, flags);
    off += (tb + 255) / 256 * 256;
  }
  L.total = off;
  return SGH_OK;
}

struct HostStreams {
  cudaStream_t in = nullptr, out = nullptr;
};
static std::mutex g_hs_mu;
static std::map<int, HostStreams> g_hs;

static sgh_status get_streams(HostStreams &hs) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_hs_mu);
  HostStreams &h = g_hs[dev];
  if (!h.in) {
    if ((e = cudaStreamCreateWithFlags(&h.in, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
    if ((e = cudaStreamCreateWithFlags(&h.out, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
  }
  hs = h;
  return SGH_OK;
}

}  // namespace sgh

using namespace sgh;

extern "C" {

size_t sgh_batched_host_buffer_bytes(const int32_t *levels, int32_t d, int64_t num_grids, uint32_t flags) {
  return guarded_value<size_t>(0, [&]() -> size_t {
  if (!levels || num_grids <= 0) return 0;
  HostLayout L;
  if (host_layout(levels, d, num_grids, flags, L) != SGH_OK)
    return 0;
  return L.total;
});
}

sgh_status sgh_transform_batched_host(double *const *host_grids, const int32_t *levels, int32_t d,
                                      int64_t num_grids, uint32_t flags, void *device_buffer,
                                      size_t device_buffer_bytes, void *stream) {
  return guarded([&]() -> sgh_status {
  if (flags & ~kKnownFlags) return invalid("unknown flags");
  if (num_grids < 0) return invalid("num_grids < 0");
  if (num_grids == 0) return SGH_OK;
  if (!host_grids || !levels) return invalid("NULL argument");
  for (int64_t g = 0; g < num_grids; ++g)
    if (!host_grids[g]) return invalid("host_grids[g] is NULL");
  HostLayout L;
  sgh_status st = host_layout(levels, d, num_grids, flags, L);
  if (st != SGH_OK) return st;
  if (!device_buffer || device_buffer_bytes < L.total || (reinterpret_cast<uintptr_t>(device_buffer) & 255)) {
    set_error("device_buffer missing, misaligned or smaller than sgh_batched_host_buffer_bytes()");
    return SGH_ERR_WORKSPACE;
  }
  HostStreams hs;
  if ((st = get_streams(hs)) != SGH_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned char *base = static_cast<unsigned char *>(device_buffer);
  // Device placement: a grid whose host memory directly follows the previous
  // grid's is placed directly after it on the device too, so a run of
  // host-contiguous grids moves with ONE copy per direction (exactly the
  // grids' own bytes: no memory between them is touched); other grids start
  // 256-byte aligned.  Offsets never exceed the padded layout of host_layout.
  std::vector<double *> dptr(num_grids);
  std::vector<int64_t> N(num_grids);
  std::vector<char> cont(num_grids, 0);              // host-contiguous with grid g - 1
  size_t off = 0;
  for (int64_t g = 0; g < num_grids; ++g) {
    validate_levels(levels + g * d, d, &N[g]);
    cont[g] = g > 0 && host_grids[g] == host_grids[g - 1] + N[g - 1];
    if (!cont[g]) off = (off + 255) / 256 * 256;
    dptr[g] = reinterpret_cast<double *>(base + off);
    off += size_t(N[g]) * 8;
  }
  cudaError_t e;
  cudaEvent_t ev_start;
  if ((e = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "event");
  cudaEventRecord(ev_start, s);
  cudaStreamWaitEvent(hs.in, ev_start, 0);
  cudaStreamWaitEvent(hs.out, ev_start, 0);
  cudaEventDestroy(ev_start);
  cudaEvent_t last_out = nullptr;
  for (size_t c = 0; c < L.chunks.size(); ++c) {
    const int64_t g0 = L.chunks[c].first, g1 = L.chunks[c].second;
    auto copy_runs = [&](bool h2d) -> cudaError_t {
      for (int64_t g = g0; g < g1;) {
        int64_t h = g + 1;
        size_t bytes = size_t(N[g]) * 8;
        while (h < g1 && cont[h]) bytes += size_t(N[h++]) * 8;
        cudaError_t ce = h2d ? cudaMemcpyAsync(dptr[g], host_grids[g], bytes, cudaMemcpyHostToDevice, hs.in)
                             : cudaMemcpyAsync(host_grids[g], dptr[g], bytes, cudaMemcpyDeviceToHost, hs.out);
        if (ce != cudaSuccess) return ce;
        g = h;
      }
      return cudaSuccess;
    };
    if ((e = copy_runs(true)) != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
    cudaEvent_t ev_in, ev_comp, ev_out;
    cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_comp, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming);
    cudaEventRecord(ev_in, hs.in);
    cudaStreamWaitEvent(s, ev_in, 0);
    void *ws = base + L.table_off[c];
    const size_t ws_bytes = (c + 1 < L.table_off.size() ? L.table_off[c + 1] : L.total) - L.table_off[c];
    st = run_batched(dptr.data() + g0, levels + g0 * d, d, g1 - g0, flags, ws, ws_bytes, s);
    if (st != SGH_OK) return st;
    cudaEventRecord(ev_comp, s);
    cudaStreamWaitEvent(hs.out, ev_comp, 0);
    if ((e = copy_runs(false)) != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync D2H");
    cudaEventRecord(ev_out, hs.out);
    cudaEventDestroy(ev_in);
    cudaEventDestroy(ev_comp);
    if (last_out) cudaEventDestroy(last_out);
    last_out = ev_out;
  }
  if (last_out) {
    cudaStreamWaitEvent(s, last_out, 0);
    cudaEventDestroy(last_out);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "e2e batched");
  return SGH_OK;
});
}

}  // extern "C"
