// sgh_plan.hpp -- host-side planning of per-axis passes into kernel phases.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "../../include/sgh.h"
#include "sgh_common.cuh"

namespace sgh {

// launchers (sgh_kernels.cu)
cudaError_t launch_single(const Task &task, bool inv, cudaStream_t stream);
cudaError_t launch_table(int kind, int l, int w, bool inv, const Task *d_tasks, const int64_t *d_prefix,
                         int32_t ntasks, int64_t total_tiles, size_t smem, double points, cudaStream_t stream,
                         int variant = 0, bool pipe = false);
// W == 1 FUSED tasks that run on the pipelined bulk-copy kernel k_fpipe (grouped separately)
// batched: grouped launches of the batched driver over several grids (padded
// lattice views stay on k_fused there); false: one grid's tasks
bool pipe_task(const Task &t, bool batched = false);
size_t task_smem(const Task &t);

// per-launch profiling (sgh_profile.cu); a no-op unless sgh_profile_enable(1)
struct ProfToken {
  cudaEvent_t start;
};
ProfToken prof_begin(cudaStream_t s);
// variant: 0 dense / per-axis, 1 BLOCKED fused tiles, 2 coarse-lattice views of a
// blocked group, 3 a grouped launch mixing 1 and 2
void prof_end(ProfToken tok, int kind, int l, bool inv, double bytes, cudaStream_t s, int variant = 0);
bool prof_active();                   // per-launch profiling on (sgh_profile_enable(1))
inline int task_variant(const Task &t) {
  if (t.kind != KIND_FUSED || t.bj < 0) return 0;
  return t.bt < t.gl[t.bj] ? 1 : 2;
}

// points a task transforms (= writes): 16 B each is its algorithmic traffic
inline double task_points(const Task &t) {
  if (t.kind == KIND_FUSED) {
    if (t.bj >= 0 && t.bt < t.gl[t.bj]) {           // blocked: the fine points of every block
      const int lj = t.gl[t.bj];
      const double fine = double((int64_t(1) << lj) - 1) - double((int64_t(1) << (lj - t.bt)) - 1);
      if (t.bt2 >= 0) {                             // two blocked axes: fine along both
        const double fine2 = double(int64_t(1) << t.nb2_log) * double((int64_t(1) << t.bt2) - 1);
        return double(t.O) * double(t.S) * double(t.P / t.ej / ((1 << t.bt2) + 1)) * fine * fine2;
      }
      return double(t.O) * double(t.S) * double(t.P / t.ej) * fine;
    }
    if (t.bj >= 0 && t.bt2 >= 0) {                 // lattice axis x blocked axis: fine rows of the latter
      const double fine2 = double(int64_t(1) << t.nb2_log) * double((int64_t(1) << t.bt2) - 1);
      return double(t.O) * double(t.S) * double(t.P / ((1 << t.bt2) + 1)) * fine2;
    }
    return double(t.O) * double(t.P) * double(t.S);   // every point, once
  }
  const int64_t n = (int64_t(1) << t.l) - 1;
  const int64_t coarse = (t.t < t.l) ? (int64_t(1) << (t.l - t.t)) - 1 : 0;
  return double(t.O) * double(t.S) * double(n - coarse);
}

// error bookkeeping (sgh_capi.cu)
void set_error(const std::string &msg);
void count_launch(uint64_t k = 1);

// Phases of one pole view in HIERARCHIZATION order (block tiles first, then
// the coarse lattice).  Dehierarchization runs them in reverse order.
void plan_view(double *grid, int64_t O, int64_t OS, int64_t PS, int64_t S, int64_t base, int l,
               std::vector<Task> &phases);

// Phases of the axis-k pass (0-based) of a grid with level vector levels[0..d).
// rows_last >= 0 overrides the extent of the last axis (a row shard of the
// grid, sharded path); then k must be < d-1.
void plan_axis(double *grid, const int32_t *levels, int d, int k, std::vector<Task> &phases,
               int64_t rows_last = -1);

// Only the fine part (tz(i) < tb) of a pole view: one FLAT_BLOCKS / STRIDED
// phase over all 2^{l-tb} blocks (rlog = l - tb, blk0 = 0).  False if no tile fits.
bool plan_view_fine(double *grid, int64_t O, int64_t OS, int64_t PS, int64_t S, int64_t base, int l, int tb,
                    std::vector<Task> &phases);

// No C++ exception may cross the C ABI (sgh.h): every extern "C" entry point
// that builds host containers runs its body through one of these.  Host
// allocation failure -> SGH_ERR_CAPACITY, anything else -> INVALID_ARGUMENT,
// with the detail in sgh_last_error().
template <class F>
sgh_status guarded(F &&body) {
  try {
    return body();
  } catch (const std::bad_alloc &) {
    set_error("host allocation failed (request too large)");
    return SGH_ERR_CAPACITY;
  } catch (const std::exception &e) {
    set_error(std::string("internal error: ") + e.what());
    return SGH_ERR_INVALID_ARGUMENT;
  } catch (...) {
    set_error("internal error");
    return SGH_ERR_INVALID_ARGUMENT;
  }
}
// the same for entry points that return a size / count (`fail` on error)
template <class T, class F>
T guarded_value(T fail, F &&body) {
  try {
    return body();
  } catch (const std::bad_alloc &) {
    set_error("host allocation failed (request too large)");
  } catch (const std::exception &e) {
    set_error(std::string("internal error: ") + e.what());
  } catch (...) {
    set_error("internal error");
  }
  return fail;
}

// helpers shared by the drivers (sgh_capi.cu)
sgh_status cuda_fail(cudaError_t e, const char *where);
sgh_status invalid(const char *msg);
sgh_status validate_levels(const int32_t *levels, int32_t d, int64_t *N_out);
sgh_status staged_upload(void *dst, const void *src, size_t bytes, cudaStream_t stream);
// batched driver: transform num_grids grids whose task tables go to `workspace`
sgh_status run_batched(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids,
                       uint32_t flags, void *workspace, size_t ws_bytes, cudaStream_t s);
size_t batched_table_bytes(double *const *grids, const int32_t *levels, int32_t d, int64_t num_grids,
                           uint32_t flags);
// flags: SGH_FLAG_DEHIERARCHIZE / SGH_FLAG_PER_AXIS / SGH_FLAG_WHOLE_POLES (sgh.h)
void plan_grid(double *grid, const int32_t *levels, int d, uint32_t flags, std::vector<std::vector<Task>> &passes);
// halo-sharded hierarchization of rank r's row shard as one box plan (the
// interior of super-block r of level T of x_d fused with the other axes)
bool plan_shard_box(double *shard, const int32_t *levels, int d, int T, int64_t r, std::vector<Task> &phases);
// plan_grid of `outer` stacked copies of the grid (a row shard of the next axis)
void plan_grid_rows(double *grid, const int32_t *levels, int d, int64_t outer, uint32_t flags,
                    std::vector<std::vector<Task>> &passes);
constexpr uint32_t kKnownFlags =
    SGH_FLAG_DEHIERARCHIZE | SGH_FLAG_PER_AXIS | SGH_FLAG_WHOLE_POLES | SGH_FLAG_TWO_BLOCKED | SGH_FLAG_TABLE_RESIDENT;
// flags that select the plan (the plan cache key)
constexpr uint32_t kPlanFlags = kKnownFlags & ~uint32_t(SGH_FLAG_TABLE_RESIDENT);

// Tuning knobs (experiments only): read from the environment in a -DSGH_TUNING
// build, compile-time defaults otherwise -- the default library reads no
// environment variable.
#ifdef SGH_TUNING
#include <cstdlib>
inline const char *tuning_env(const char *name) { return std::getenv(name); }
#else
inline const char *tuning_env(const char *) { return nullptr; }
#endif

}  // namespace sgh
