// C ABI of libdifftrans (include/difftrans.h): argument checking, context-owned memory,
// the record-arena policy and the per-depth launch sequence.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "dt_internal.h"

using namespace dt;

namespace {

dt_status fail(dt_ctx* c, dt_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define DT_CU(call)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) {                                                                     \
      dt_status s_ = e_ == cudaErrorMemoryAllocation ? DT_ERR_OOM : DT_ERR_CUDA;                 \
      return fail(c, s_, "%s failed: %s", #call, cudaGetErrorString(e_));                        \
    }                                                                                            \
  } while (0)

#define DT_ARG(cond, ...) \
  do {                    \
    if (!(cond)) return fail(c, DT_ERR_INVALID_ARG, __VA_ARGS__); \
  } while (0)

cudaError_t alloc_arena(dt_ctx* c, int64_t cap) {
  if (c->rec.o) cudaFree(c->rec.o);
  c->rec = Records{};
  c->arena_cap = 0;
  char* base = nullptr;
  const size_t bytes = (size_t)cap * (kRecordBytes + (c->arena_vol ? 32 : 0));
  cudaError_t e = cudaMalloc(&base, bytes);
  if (e != cudaSuccess) return e;
  c->rec.o = reinterpret_cast<Vec64*>(base);
  c->rec.d = c->rec.o + cap;
  float4* f = reinterpret_cast<float4*>(c->rec.d + cap);
  c->rec.thr = f;
  c->rec.hit = f + cap;
  c->rec.tau = f + 2 * cap;
  c->rec.lsub = f + 3 * cap;
  c->rec.go = f + 4 * cap;
  c->rec.gd = f + 5 * cap;
  if (c->arena_vol) {
    c->rec.mq = f + 6 * cap;
    c->rec.mg = f + 7 * cap;
  }
  c->arena_cap = cap;
  return cudaSuccess;
}

// Absorption parameter block checks and sizes (R11, R29).
bool abs_valid(const dt_absorption* ab) {
  if (ab->kind == DT_ABS_CONST) return true;
  if (ab->n_samples < 1) return false;
  if (ab->kind == DT_ABS_GRID) return ab->res >= 2;
  if (ab->kind != DT_ABS_HASH || ab->levels < 1 || ab->levels > 32 || ab->log2_size < 1 || ab->log2_size > 26)
    return false;
  for (int l = 0; l < ab->levels; ++l)
    if (ab->level_res[l] < 1 || ab->level_res[l] > (1 << 20)) return false;
  return true;
}

size_t abs_nodes(const dt_absorption* ab) {
  if (ab->kind == DT_ABS_CONST) return 1;
  if (ab->kind == DT_ABS_HASH) return (size_t)ab->levels << ab->log2_size;
  return (size_t)ab->res * ab->res * ab->res;
}

int64_t arena_limit(const dt_ctx* c) {
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  return (int64_t)((double)fr * 0.70 / (kRecordBytes + (c->arena_vol ? 32 : 0)));
}

cudaEvent_t get_event(dt_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Fold completed phase timings into the totals (waits on the pending events).
// block = false: only fold the events that have already completed (never stalls the host
// behind queued GPU work, so an asynchronous step loop keeps the GPU fed).
void resolve_profile(dt_ctx* c, bool block = true) {
  size_t i = 0;
  for (; i < c->pending.size(); ++i) {
    auto& p = c->pending[i];
    if (block) cudaEventSynchronize(p.b);
    else if (cudaEventQuery(p.b) != cudaSuccess) break;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) c->ph_ms[p.ph] += ms;
    c->event_pool.push_back(p.a);
    c->event_pool.push_back(p.b);
  }
  c->pending.erase(c->pending.begin(), c->pending.begin() + i);
}

// Records needed by a forward with level counts `lvl` (attempted appends; levels after an
// overflow were not run and are extrapolated with the last known level size).
int64_t level_need(const int* lvl, int D) {
  int64_t need = 0, last = 0;
  int known = 0;
  for (int k = 0; k <= D; ++k) {
    int64_t v = (unsigned)lvl[LV_CNT + k];
    if (v == 0 && k > 0) break;
    need += v;
    last = v;
    known = k;
  }
  return need + last * (D - known);
}

void fill_stats(dt_ctx* c, dt_stats* st) {
  memset(st, 0, sizeof(*st));
  const int* h = c->host_lvl;
  int64_t seg = h[LV_TRACED];
  for (int k = 0; k <= c->last_D; ++k) {
    st->segments_per_depth[k] = h[LV_CNT + k];
    if (k > 0) seg += h[LV_CNT + k];
  }
  st->primaries = c->last_rays;
  st->primaries_traced = h[LV_TRACED];
  st->segments = seg;
  st->arena_capacity = c->arena_cap;
  st->arena_retries = c->last_retries;
}

}  // namespace

// Check a pending asynchronous forward: wait for its readback, record its need, and report
// an overflow (growing the arena for the next step).
dt_status consume_async(dt_ctx* c) {
  if (!c->async_pending && !c->graph_fwd) return DT_OK;
  if (c->async_pending) {
    cudaError_t e = cudaEventSynchronize(c->fwd_done);
    if (e != cudaSuccess) return fail(c, DT_ERR_CUDA, "async forward: %s", cudaGetErrorString(e));
  }
  // (graph replays: the caller has synchronised the replay stream; host_lvl is the last replay's)
  c->async_pending = false;
  if (c->prof) resolve_profile(c, false);
  int64_t need = level_need(c->host_lvl, c->last_D);
  c->last_need = need;
  if (c->host_lvl[LV_STACKERR]) return fail(c, DT_ERR_STACK, "async forward: BVH deeper than the traversal stack");
  if (c->host_lvl[LV_OVERFLOW]) {
    int64_t next = std::min<int64_t>(need + need / 2 + 65536, arena_limit(c) + c->arena_cap);
    if (next > c->arena_cap && alloc_arena(c, next) != cudaSuccess)
      return fail(c, DT_ERR_OOM, "async forward overflowed and the arena could not grow to %lld", (long long)next);
    c->have_fwd = false;
    return fail(c, DT_ERR_RETRY, "the previous asynchronous forward overflowed the record arena (need %lld); "
                "re-run that step", (long long)need);
  }
  return DT_OK;
}

PhaseTimer::PhaseTimer(dt_ctx* c_, int ph_, cudaStream_t st_) : c(c_), ph(ph_), st(st_) {
  if (c->prof) {
    a = get_event(c);
    cudaEventRecord(a, st);
  }
}

void PhaseTimer::end(int n_launches) {
  c->ph_launches[ph] += n_launches;
  c->kernel_launches += n_launches;
  if (c->prof) {
    cudaEvent_t b = get_event(c);
    cudaEventRecord(b, st);
    c->pending.push_back({ph, a, b});
  }
}

namespace dt {
DT_DEFINE_CHECK_READER(check_status_api)
}  // namespace dt

extern "C" {

const char* dt_status_string(dt_status s) {
  switch (s) {
    case DT_OK: return "DT_OK";
    case DT_ERR_INVALID_ARG: return "DT_ERR_INVALID_ARG";
    case DT_ERR_EMPTY_GEOMETRY: return "DT_ERR_EMPTY_GEOMETRY";
    case DT_ERR_CUDA: return "DT_ERR_CUDA";
    case DT_ERR_OOM: return "DT_ERR_OOM";
    case DT_ERR_NOT_BUILT: return "DT_ERR_NOT_BUILT";
    case DT_ERR_NO_FORWARD: return "DT_ERR_NO_FORWARD";
    case DT_ERR_NONFINITE: return "DT_ERR_NONFINITE";
    case DT_ERR_STACK: return "DT_ERR_STACK";
    case DT_ERR_RETRY: return "DT_ERR_RETRY";
  }
  return "DT_ERR_UNKNOWN";
}

dt_status dt_create(int32_t device, dt_ctx** out) {
  dt_ctx* c = nullptr;
  if (!out) return DT_ERR_INVALID_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return DT_ERR_CUDA;
  if (device < 0 || device >= n) return DT_ERR_INVALID_ARG;
  c = new dt_ctx();
  c->device = device;
  cudaSetDevice(device);
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e;
  if ((e = cudaMalloc(&c->lvl, LV_INTS * sizeof(int))) || (e = cudaMallocHost(&c->host_lvl, LV_INTS * sizeof(int))) ||
      (e = cudaMalloc(&c->gior, 4 * sizeof(float))) || (e = cudaMalloc(&c->counters, 8 * sizeof(unsigned long long))) ||
      (e = cudaMemset(c->counters, 0, 8 * sizeof(unsigned long long))) ||
      (e = cudaEventCreateWithFlags(&c->fwd_done, cudaEventDisableTiming)) ||
      (e = cudaMalloc(&c->scratch, 16 * sizeof(unsigned)))) {
    dt_destroy(c);
    return e == cudaErrorMemoryAllocation ? DT_ERR_OOM : DT_ERR_CUDA;
  }
  *out = c;
  return DT_OK;
}

void dt_destroy(dt_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  void* ptrs[] = {c->V, c->F, c->nrm, c->fnrm, c->nodes, c->tris, c->keys, c->vals, c->hist, c->children,
                  c->parent_int, c->parent_leaf, c->rflags, c->nodebox, c->leafbox, c->vstart, c->vcorner, c->scal,
                  c->iscal, c->rec.o, c->lvl, c->sigma_snap, c->gV, c->gN, c->gVn, c->gS, c->fe, c->gsig, c->gior,
                  c->counters, c->ranges, c->wbox, c->wdepth, c->went, c->scratch,
                  c->nbr_start, c->nbr_cnt, c->nbr, c->nbr_owner, c->scan_part, c->wqueue};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& p : c->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->host_lvl) cudaFreeHost(c->host_lvl);
  if (c->fwd_done) cudaEventDestroy(c->fwd_done);
  delete c;
}

const char* dt_last_error(const dt_ctx* c) { return c ? c->err.c_str() : "null context"; }

const int32_t* dt_forward_overflow_flag(const dt_ctx* c) { return c ? c->lvl + LV_OVERFLOW : nullptr; }

dt_status dt_build_bvh(dt_ctx* c, const float* V, int32_t nv, const int32_t* F, int32_t nf, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (nv <= 0 || nf <= 0) return fail(c, DT_ERR_EMPTY_GEOMETRY, "dt_build_bvh: empty geometry (nv=%d, nf=%d)", nv, nf);
  DT_ARG(V && F, "dt_build_bvh: V and F must be non-NULL device pointers");
  DT_ARG(nf < (1 << 29) && nv < (1 << 29), "dt_build_bvh: nv/nf too large");
  cudaStream_t st = (cudaStream_t)stream;
  PhaseTimer pt(c, DT_PH_BUILD, st);
  int nl = 0;
  DT_CU(build_bvh(c, V, nv, F, nf, st, &nl));
  pt.end(nl);
  c->built = true;
  c->have_fwd = false;
  return DT_OK;
}

dt_status dt_set_bvh_quality(dt_ctx* c, int32_t treelet_passes) {
  if (!c) return DT_ERR_INVALID_ARG;
  DT_ARG(treelet_passes >= 0 && treelet_passes <= 4, "dt_set_bvh_quality: treelet_passes=%d not in [0, 4]",
         treelet_passes);
  c->treelet_passes = treelet_passes;
  return DT_OK;
}

dt_status dt_trace_forward(dt_ctx* c, float ior, const dt_absorption* ab, const dt_env* env, const dt_cameras* cams,
                           const dt_trace_opts* opts, float* rgb, float* capped_w, uint64_t* sig_topo,
                           uint64_t* sig_face, dt_stats* stats, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (!c->built) return fail(c, DT_ERR_NOT_BUILT, "dt_trace_forward: call dt_build_bvh first");
  DT_ARG(ab && env && cams && opts, "dt_trace_forward: absorption/env/cams/opts must be non-NULL");
  DT_ARG(opts->max_depth >= 0 && opts->max_depth <= DT_MAX_DEPTH, "dt_trace_forward: opts.max_depth=%d not in [0,%d]",
         opts->max_depth, DT_MAX_DEPTH);
  DT_ARG(opts->cap_policy == DT_CAP_ZERO || opts->cap_policy == DT_CAP_ENV, "dt_trace_forward: bad opts.cap_policy");
  DT_ARG(opts->t_eps >= 0.0f, "dt_trace_forward: opts.t_eps must be >= 0");
  DT_ARG(ior > 0.0f, "dt_trace_forward: ior must be > 0");
  DT_ARG(cams->K && cams->c2w && cams->n_views > 0 && cams->width > 0 && cams->height > 0,
         "dt_trace_forward: cams (K, c2w, n_views, width, height) invalid");
  DT_ARG(ab->sigma, "dt_trace_forward: absorption.sigma is NULL");
  DT_ARG(abs_valid(ab), "dt_trace_forward: absorption (kind=%d res=%d n_samples=%d levels=%d log2_size=%d) invalid",
         ab->kind, ab->res, ab->n_samples, ab->levels, ab->log2_size);
  DT_ARG((env->kind == DT_ENV_ANALYTIC && (env->n_lobes == 0 || env->lobes)) ||
             ((env->kind == DT_ENV_GRID || env->kind == DT_ENV_VOLUME) && env->voxel && env->planes && env->vres >= 2 &&
              env->pres >= 2 && env->radius > 0 &&
              (env->kind == DT_ENV_GRID || (env->n_samples >= 1 && !env->far_field))),
         "dt_trace_forward: env (kind=%d) invalid", env->kind);
  int64_t npix = (int64_t)cams->n_views * cams->width * cams->height;
  const bool tiled = !cams->pixel_ids && cams->tile > 0;
  int64_t n_rays = cams->pixel_ids ? cams->n_rays : npix;
  if (tiled) {
    DT_ARG(cams->tile % 8 == 0 && cams->width % cams->tile == 0 && cams->height % cams->tile == 0,
           "dt_trace_forward: tile=%d must be a multiple of 8 dividing width %d and height %d", cams->tile,
           cams->width, cams->height);
    const int64_t total = npix / ((int64_t)cams->tile * cams->tile);
    int64_t nt;
    if (cams->tile_ids) {
      DT_ARG(cams->n_tiles >= 0, "dt_trace_forward: n_tiles < 0");
      nt = cams->n_tiles;
    } else {
      DT_ARG(cams->shard_count >= 1 && cams->shard_rank >= 0 && cams->shard_rank < cams->shard_count,
             "dt_trace_forward: shard_rank %d / shard_count %d invalid", cams->shard_rank, cams->shard_count);
      nt = total > cams->shard_rank ? (total - cams->shard_rank + cams->shard_count - 1) / cams->shard_count : 0;
    }
    n_rays = nt * cams->tile * cams->tile;
  }
  DT_ARG(n_rays >= 0 && n_rays < (1ll << 31), "dt_trace_forward: n_rays=%lld out of range", (long long)n_rays);
  DT_ARG(rgb || n_rays == 0, "dt_trace_forward: rgb must be a device pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int D = opts->max_depth;
  // CUDA-graph capture (see dt_get_stats): no host synchronisation and no allocation allowed
  cudaStreamCaptureStatus cap_state = cudaStreamCaptureStatusNone;
  DT_CU(cudaStreamIsCapturing(st, &cap_state));
  const bool capturing = cap_state != cudaStreamCaptureStatusNone;
  if (capturing) {
    DT_ARG(!c->async_pending, "dt_trace_forward (capture): check the previous asynchronous forward (dt_get_stats) "
           "before capturing");
    DT_ARG(!c->prof, "dt_trace_forward (capture): profiling must be off");
    DT_ARG(opts->async && !stats && !opts->check_finite,
           "dt_trace_forward (capture): the forward must be asynchronous, without stats / check_finite");
    DT_ARG(c->last_need > 0 && c->last_rays == n_rays && c->arena_cap >= c->last_need + c->last_need / 4 &&
               abs_nodes(ab) <= c->sigma_cap && (env->kind != DT_ENV_VOLUME || c->arena_vol),
           "dt_trace_forward (capture): warm up first (an asynchronous forward of the same %lld rays, checked)",
           (long long)n_rays);
  }

  // absorption snapshot (the backward differentiates w.r.t. these values)
  size_t nodes = abs_nodes(ab);
  size_t slen = nodes * 3;
  if (nodes > c->sigma_cap) {
    if (c->sigma_snap) cudaFree(c->sigma_snap);
    if (c->gsig) cudaFree(c->gsig);
    c->sigma_snap = c->gsig = nullptr;
    c->sigma_cap = 0;
    DT_CU(cudaMalloc(&c->sigma_snap, 2 * nodes * sizeof(float4)));
    DT_CU(cudaMalloc(&c->gsig, nodes * sizeof(float4)));
    c->sigma_cap = nodes;
  }
  c->sigma_len = slen;
  // grid: x-pairs (32 B per node); constant / hash: one float4 per node / table entry
  DT_CU(launch_pack_sigma(ab->sigma, c->sigma_snap, (int64_t)nodes, ab->kind == DT_ABS_GRID ? ab->res : 1,
                          ab->kind == DT_ABS_GRID, st));

  DevScene s = scene_from_ctx(c);
  s.ior = ior;
  s.ior_ptr = opts->ior_device;
  s.abs_kind = ab->kind;
  s.sigma = c->sigma_snap;
  s.sres = ab->res;
  s.nsamp = std::max(1, ab->n_samples);
  s.slo = f3(ab->box_lo[0], ab->box_lo[1], ab->box_lo[2]);
  s.shi = f3(ab->box_hi[0], ab->box_hi[1], ab->box_hi[2]);
  if (ab->kind == DT_ABS_HASH) {
    s.hlevels = ab->levels;
    s.hlog2 = ab->log2_size;
    s.hdense = 0u;
    for (int l = 0; l < ab->levels; ++l) {
      s.hres[l] = ab->level_res[l];
      const double n1 = ab->level_res[l] + 1.0;
      if (n1 * n1 * n1 <= (double)(1u << ab->log2_size)) s.hdense |= 1u << l;
    }
  }
  s.env_kind = env->kind;
  s.ambient = f3(env->ambient[0], env->ambient[1], env->ambient[2]);
  s.lobes = env->lobes;
  s.nlobes = env->n_lobes;
  s.voxel = (const float4*)env->voxel;
  s.vres = env->vres;
  s.planes = (const float4*)env->planes;
  s.env_nsamp = env->kind == DT_ENV_VOLUME ? env->n_samples : 0;
  s.pres = env->pres;
  s.radius = env->radius;
  s.far_field = env->far_field;
  s.max_depth = D;
  s.cap_policy = opts->cap_policy;

  FwdLaunch a{};
  a.s = s;
  a.lvl = c->lvl;
  a.t_eps = opts->t_eps;
  a.K = cams->K;
  a.c2w = cams->c2w;
  a.W = cams->width;
  a.H = cams->height;
  a.n_views = cams->n_views;
  a.pids = cams->pixel_ids;
  a.tiles_x = (cams->width + 7) / 8;
  a.tiles_per_view = a.tiles_x * ((cams->height + 3) / 4);
  a.n_items = cams->pixel_ids || tiled ? n_rays : (int64_t)a.tiles_per_view * cams->n_views * 32;
  a.shard_tile = tiled ? cams->tile : 0;
  if (tiled) {
    a.stiles_x = cams->width / cams->tile;
    a.stiles_per_view = a.stiles_x * (cams->height / cams->tile);
    a.shard_rank = cams->shard_rank;
    a.shard_count = std::max(cams->shard_count, 1);
    a.tile_ids = cams->tile_ids;
  }
  a.rgb = rgb;
  a.capw = capped_w;
  a.sig_t = (unsigned long long*)sig_topo;
  a.sig_f = (unsigned long long*)sig_face;
  a.counters = c->counters;
  a.grids = c->grid_cache;
  a.segc = opts->seg_count;

  // a previous asynchronous forward is checked first (its readback has long completed)
  dt_status prev = capturing ? DT_OK : consume_async(c);
  if (!capturing) c->graph_fwd = false;   // an eager forward replaces the captured one's state
  if (prev != DT_OK) return prev;
  int64_t limit = 0;   // HBM budget, queried (cudaMemGetInfo) only when the arena must grow
  if (env->kind == DT_ENV_VOLUME && !c->arena_vol) {   // the volume needs two more record lanes
    c->arena_vol = true;
    if (c->arena_cap > 0) DT_CU(alloc_arena(c, c->arena_cap));
  }
  if (c->arena_cap == 0) {
    limit = arena_limit(c);
    int64_t want = std::min<int64_t>(std::max<int64_t>(n_rays * 3, 1 << 16), limit);
    DT_CU(alloc_arena(c, want));
  }
  bool async = opts->async && !stats && !opts->check_finite && c->last_need > 0 && c->last_rays == n_rays;
  if (async && c->arena_cap < c->last_need + c->last_need / 4) {   // keep 25% headroom
    limit = arena_limit(c) + c->arena_cap;
    int64_t next = std::min<int64_t>(c->last_need + c->last_need / 2 + 65536, limit);
    if (next > c->arena_cap) DT_CU(alloc_arena(c, next));
    async = c->arena_cap >= c->last_need + c->last_need / 4;
  }
  int retries = 0;
  while (true) {
    a.r = c->rec;
    a.cap = c->arena_cap;
    DT_CU(cudaMemsetAsync(c->lvl, 0, LV_INTS * sizeof(int), st));
    if (capped_w) DT_CU(cudaMemsetAsync(capped_w, 0, (size_t)n_rays * sizeof(float), st));
    if (sig_topo) DT_CU(cudaMemsetAsync(sig_topo, 0, (size_t)n_rays * sizeof(uint64_t), st));
    if (sig_face) DT_CU(cudaMemsetAsync(sig_face, 0, (size_t)n_rays * sizeof(uint64_t), st));
    if (n_rays > 0) {
      {
        PhaseTimer p(c, DT_PH_TRACE0, st);
        DT_CU(launch_trace_primary(a, D, c->sm_count, st));
        p.end(1);
      }
      {
        PhaseTimer p(c, DT_PH_SHADE, st);
        DT_CU(launch_shade_level(a, 0, D, c->sm_count, st));
        p.end(1);
      }
      for (int k = 1; k <= D; ++k) {
        {
          PhaseTimer p(c, DT_PH_TRACE, st);
          DT_CU(launch_traverse_level(a, k, c->sm_count, st));
          p.end(1);
        }
        PhaseTimer p(c, DT_PH_SHADE, st);
        DT_CU(launch_shade_level(a, k, D, c->sm_count, st));
        p.end(1);
      }
      for (int k = std::max(D - 1, 0); k >= 0; --k) {
        PhaseTimer p(c, DT_PH_GATHER, st);
        DT_CU(launch_gather_level(a, k, c->sm_count, st));
        p.end(1);
      }
    }
    DT_CU(launch_count_segments(c->lvl, D, c->counters + 4, st));
    c->kernel_launches += 1;
    DT_CU(cudaMemcpyAsync(c->host_lvl, c->lvl, LV_INTS * sizeof(int), cudaMemcpyDeviceToHost, st));
    c->last_D = D;
    c->last_rays = n_rays;
    c->last_retries = retries;
    if (async) {
      if (capturing) {
        c->graph_fwd = true;           // host_lvl refreshed by every replay (the copy above)
      } else {
        DT_CU(cudaEventRecord(c->fwd_done, st));
        c->async_pending = true;
      }
      break;
    }
    DT_CU(cudaStreamSynchronize(st));
    if (!c->host_lvl[LV_OVERFLOW]) break;
    int64_t need = level_need(c->host_lvl, D);
    int64_t next = std::max<int64_t>(c->arena_cap + c->arena_cap / 4, need + need / 8 + 65536);
    limit = arena_limit(c) + c->arena_cap;
    if (c->arena_cap >= limit || ++retries > 8)
      return fail(c, DT_ERR_OOM, "dt_trace_forward: record arena needs > %lld records (HBM budget %lld)",
                  (long long)next, (long long)limit);
    next = std::min(next, limit);
    DT_CU(alloc_arena(c, next));
  }
  c->have_fwd = true;
  c->n_rays = n_rays;
  c->fwd_scene = s;
  c->fwd_t_eps = opts->t_eps;
  if (async) return DT_OK;
  c->last_need = level_need(c->host_lvl, D);
  if (c->prof) resolve_profile(c);   // all recorded events are complete after the sync
  if (c->host_lvl[LV_STACKERR]) return fail(c, DT_ERR_STACK, "dt_trace_forward: BVH deeper than the traversal stack");
  if (opts->check_finite && n_rays > 0) {
    DT_CU(cudaMemsetAsync(c->lvl + LV_NONFINITE, 0, sizeof(int), st));
    DT_CU(launch_check_finite(rgb, 3 * n_rays, c->lvl + LV_NONFINITE, st));
    int flag = 0;
    DT_CU(cudaMemcpyAsync(&flag, c->lvl + LV_NONFINITE, sizeof(int), cudaMemcpyDeviceToHost, st));
    DT_CU(cudaStreamSynchronize(st));
    if (flag) return fail(c, DT_ERR_NONFINITE, "dt_trace_forward: rgb has non-finite values");
  }
  if (stats) fill_stats(c, stats);
  return DT_OK;
}

dt_status dt_get_stats(dt_ctx* c, dt_stats* out) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  DT_ARG(out, "dt_get_stats: out is NULL");
  if (!c->have_fwd) return fail(c, DT_ERR_NO_FORWARD, "dt_get_stats: no forward on this context");
  dt_status prev = consume_async(c);
  fill_stats(c, out);
  return prev;
}

dt_status dt_trace_backward(dt_ctx* c, const float* grad_rgb, float* grad_V, float* grad_ior, float* grad_sigma,
                            int32_t accumulate, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (!c->have_fwd) return fail(c, DT_ERR_NO_FORWARD, "dt_trace_backward: no forward on this context");
  // an asynchronous forward is not waited for: the backward kernels skip an overflowed arena
  // on the device, and the overflow is reported by the next forward / dt_get_stats
  DT_ARG(grad_rgb || c->n_rays == 0, "dt_trace_backward: grad_rgb is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  DT_CU(cudaMemsetAsync(c->gV, 0, (size_t)c->nv * 16, st));
  DT_CU(cudaMemsetAsync(c->gN, 0, (size_t)c->nv * 16, st));
  DT_CU(cudaMemsetAsync(c->gsig, 0, (c->sigma_len / 3) * sizeof(float4), st));
  DT_CU(cudaMemsetAsync(c->gior, 0, sizeof(float), st));
  DT_CU(cudaMemsetAsync(c->lvl + LV_WORK_BWD, 0, 16 * sizeof(int), st));
  BwdLaunch b{};
  b.s = c->fwd_scene;
  b.grids = c->grid_cache;
  b.r = c->rec;
  b.lvl = c->lvl;
  b.cap = c->arena_cap;
  b.t_eps = c->fwd_t_eps;
  b.grad_rgb = grad_rgb;
  b.dV = c->gV;
  b.dN = c->gN;
  b.dsig = c->gsig;
  b.dior = c->gior;
  if (c->n_rays > 0)
    for (int k = b.s.max_depth; k >= 0; --k) {
      PhaseTimer p(c, DT_PH_BWD, st);
      DT_CU(launch_backward_level(b, k, c->sm_count, st));
      p.end(1);
    }
  PhaseTimer p(c, DT_PH_NORMALS_BWD, st);
  DT_CU(launch_vertex_normal_backward(c, st));
  DT_CU(launch_finalize(c, grad_V, grad_ior, grad_sigma, accumulate, st));
  p.end(3 + (grad_V ? 1 : 0) + (grad_ior ? 1 : 0) + (grad_sigma ? 1 : 0));
  return DT_OK;
}

dt_status dt_set_profiling(dt_ctx* c, int32_t enable) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (!enable) resolve_profile(c);
  c->prof = enable != 0;
  return DT_OK;
}

dt_status dt_get_profile(dt_ctx* c, dt_profile* out, int32_t reset) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  DT_ARG(out, "dt_get_profile: out is NULL");
  resolve_profile(c);
  unsigned long long cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  DT_CU(cudaMemcpy(cnt, c->counters, sizeof(cnt), cudaMemcpyDeviceToHost));
  for (int i = 0; i < DT_PH_COUNT; ++i) {
    out->ms[i] = c->ph_ms[i];
    out->launches[i] = c->ph_launches[i];
  }
  out->kernel_launches = c->kernel_launches;
  out->node_visits = (int64_t)(cnt[0] + cnt[2]);
  out->tri_tests = (int64_t)(cnt[1] + cnt[3]);
  out->node_visits_primary = (int64_t)cnt[2];
  out->tri_tests_primary = (int64_t)cnt[3];
  out->segments = (int64_t)cnt[4];
  out->walk_cells_fwd = (int64_t)cnt[5];
  out->walk_cells_bwd = (int64_t)cnt[6];
  out->env_samples_bwd = (int64_t)cnt[7];
  if (reset) {
    for (int i = 0; i < DT_PH_COUNT; ++i) { c->ph_ms[i] = 0.0; c->ph_launches[i] = 0; }
    c->kernel_launches = 0;
    DT_CU(cudaMemset(c->counters, 0, sizeof(cnt)));
  }
  return DT_OK;
}

dt_status dt_loss_color(dt_ctx* c, const float* rgb, const float* target, int64_t n, float* grad_rgb, float* loss,
                        void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  DT_ARG(rgb && target && grad_rgb && loss, "dt_loss_color: NULL argument");
  DT_ARG(n >= 0, "dt_loss_color: n < 0");
  PhaseTimer p(c, DT_PH_LOSS, (cudaStream_t)stream);
  DT_CU(launch_loss_color(rgb, target, n, grad_rgb, loss, (cudaStream_t)stream));
  p.end(1);
  return DT_OK;
}

dt_status dt_loss_rt(dt_ctx* c, const float* rgb, const float* target, const float* mask, int64_t n, float lambda_color,
                     float lambda_tone, float* grad_rgb, float* loss, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  DT_ARG(loss && (n == 0 || (rgb && target && grad_rgb)), "dt_loss_rt: NULL argument");
  DT_ARG(n >= 0, "dt_loss_rt: n < 0");
  PhaseTimer p(c, DT_PH_LOSS, (cudaStream_t)stream);
  DT_CU(launch_loss_rt(rgb, target, mask, n, lambda_color, lambda_tone, grad_rgb, loss, (cudaStream_t)stream));
  p.end(n > 0 ? 1 : 0);
  return DT_OK;
}

dt_status dt_sigma_regularizers(dt_ctx* c, const dt_absorption* ab, const float* points, const float* xi, int64_t n,
                                float lambda_smooth, float lambda_vol, float* grad_sigma, float* loss, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  DT_ARG(ab && ab->sigma && grad_sigma && loss, "dt_sigma_regularizers: NULL argument");
  DT_ARG(abs_valid(ab), "dt_sigma_regularizers: bad absorption");
  DT_ARG(n >= 0 && (n == 0 || ab->kind == DT_ABS_CONST || (points && xi)), "dt_sigma_regularizers: points/xi");
  PhaseTimer p(c, DT_PH_LOSS, (cudaStream_t)stream);
  DT_CU(launch_sigma_reg(ab, points, xi, n, lambda_smooth, lambda_vol, grad_sigma, loss, (cudaStream_t)stream));
  p.end(1);
  return DT_OK;
}

dt_status dt_adam_step(dt_ctx* c, float* param, const float* grad, float* m, float* v, int64_t n, const dt_adam* cfg,
                       void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  DT_ARG(cfg && param && grad && m && v, "dt_adam_step: NULL argument");
  DT_ARG(n > 0 && (cfg->step >= 1 || cfg->step_device) && cfg->lr >= 0.f && cfg->beta1 >= 0.f && cfg->beta1 < 1.f && cfg->beta2 >= 0.f &&
             cfg->beta2 < 1.f && cfg->eps > 0.f,
         "dt_adam_step: bad configuration (n=%lld step=%d)", (long long)n, cfg->step);
  PhaseTimer p(c, DT_PH_LOSS, (cudaStream_t)stream);
  int nl = 0;
  DT_CU(launch_adam(param, grad, m, v, n, cfg, c->scratch, (cudaStream_t)stream, &nl));
  p.end(nl);
  return DT_OK;
}

dt_status dt_mesh_regularizers(dt_ctx* c, float lambda_edge, float lambda_lap, float* grad_V, float* loss,
                               void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (!c->built) return fail(c, DT_ERR_NOT_BUILT, "dt_mesh_regularizers: call dt_build_bvh first");
  DT_ARG(grad_V && loss, "dt_mesh_regularizers: grad_V and loss must be device pointers");
  DT_ARG(lambda_edge >= 0.f && lambda_lap >= 0.f, "dt_mesh_regularizers: lambdas must be >= 0");
  PhaseTimer p(c, DT_PH_LOSS, (cudaStream_t)stream);
  int nl = 0;
  DT_CU(launch_mesh_regularizers(c, lambda_edge, lambda_lap, grad_V, loss, (cudaStream_t)stream, &nl));
  p.end(nl);
  return DT_OK;
}

dt_status dt_mask_loss(dt_ctx* c, const dt_cameras* cams, const float* gt_mask, float lambda, float* grad_V,
                       float* loss, float* mask_out, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (!c->built) return fail(c, DT_ERR_NOT_BUILT, "dt_mask_loss: call dt_build_bvh first");
  DT_ARG(cams && gt_mask && grad_V && loss, "dt_mask_loss: NULL argument");
  DT_ARG(cams->K && cams->c2w && cams->n_views > 0 && cams->width > 0 && cams->height > 0 && !cams->pixel_ids &&
             cams->tile <= 0,
         "dt_mask_loss: cams must describe full images (pixel_ids = NULL, tile = 0)");
  DT_ARG(lambda >= 0.f, "dt_mask_loss: lambda must be >= 0");
  PhaseTimer p(c, DT_PH_LOSS, (cudaStream_t)stream);
  int nl = 0;
  DT_CU(launch_mask_loss(c, cams, gt_mask, lambda, grad_V, loss, mask_out, (cudaStream_t)stream, &nl));
  p.end(nl);
  return DT_OK;
}

dt_status dt_debug_closest_hit(dt_ctx* c, const float* rays, int64_t n, float t_lo, int32_t brute_force, int32_t* face,
                               float* tuv, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (!c->built) return fail(c, DT_ERR_NOT_BUILT, "dt_debug_closest_hit: call dt_build_bvh first");
  DT_ARG(rays && face && tuv, "dt_debug_closest_hit: NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  DevScene s = scene_from_ctx(c);
  DT_CU(cudaMemsetAsync(c->lvl + LV_STACKERR, 0, sizeof(int), st));
  if (n > 0) DT_CU(launch_debug_closest_hit(s, rays, n, t_lo, brute_force, face, tuv, c->lvl + LV_STACKERR, st));
  int err = 0;
  DT_CU(cudaMemcpyAsync(&err, c->lvl + LV_STACKERR, sizeof(int), cudaMemcpyDeviceToHost, st));
  DT_CU(cudaStreamSynchronize(st));
  if (err) return fail(c, DT_ERR_STACK, "dt_debug_closest_hit: traversal stack overflow");
  return DT_OK;
}

dt_status dt_debug_bvh_check(dt_ctx* c, int64_t* out, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (!c->built) return fail(c, DT_ERR_NOT_BUILT, "dt_debug_bvh_check: call dt_build_bvh first");
  DT_ARG(out, "dt_debug_bvh_check: out is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  long long* dev = nullptr;
  DT_CU(cudaMallocAsync(&dev, 4 * sizeof(long long), st));
  DT_CU(launch_bvh_check(c, dev, st));
  DT_CU(cudaMemcpyAsync(out, dev, 4 * sizeof(long long), cudaMemcpyDeviceToHost, st));
  DT_CU(cudaFreeAsync(dev, st));
  DT_CU(cudaStreamSynchronize(st));
  return DT_OK;
}

dt_status dt_debug_vertex_normals(dt_ctx* c, float* out, void* stream) {
  if (!c) return DT_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (!c->built) return fail(c, DT_ERR_NOT_BUILT, "dt_debug_vertex_normals: call dt_build_bvh first");
  DT_ARG(out, "dt_debug_vertex_normals: out is NULL");
  DT_CU(launch_normals_to_f32(c->nrm, c->nv, out, (cudaStream_t)stream));
  return DT_OK;
}

dt_status dt_debug_check_status(int32_t* out) {
  if (!out) return DT_ERR_INVALID_ARG;
  if (cudaDeviceSynchronize() != cudaSuccess) return DT_ERR_CUDA;
  out[0] = dt::check_status_bvh();
  out[1] = dt::check_status_trace();
  out[2] = dt::check_status_optim();
  out[3] = dt::check_status_meshreg();
  out[4] = dt::check_status_api();
  return DT_OK;
}

}  // extern "C"
