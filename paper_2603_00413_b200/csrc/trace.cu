// Wavefront forward trace, radiance gather and backward replay (K8-K14).
//
// Forward, level k = 0..D_max (one launch per depth, persistent warps, dynamic fetch):
//   traverse the level's rays through the LBVH (shared-memory short stack), then for each
//   hit evaluate the interface (Fresnel/Snell/TIR), the interior transmittance and append
//   the reflect/refract children to level k+1 with one warp-ballot compaction per warp.
//   Misses end in the environment lookup; hits at depth D_max are capped (R12, R13).
// Gather, level k = D_max-1..0: L_sub = tau * (R L_r + T L_t) bottom-up; level 0 writes
//   the pixel radiance (deterministic, no atomics).
// Backward, level k = D_max..0: local VJP per record at fixed topology; children pass
//   dL/d(origin, direction) up through their own record slots; vertex-position and
//   vertex-normal adjoints scatter with float4 atomics, IOR / constant-sigma adjoints are
//   reduced per warp.
//
// Arena layout: level 0 (camera-ray hits) grows DOWN from the top of the arena
// (record cap-1-i), levels 1..D_max are contiguous from the bottom (level k starts at
// sum_{1<=j<k} cnt_j).  So every level's start is known once the previous level is done.
#include <cuda_runtime.h>

#include <algorithm>

#include "dt_internal.h"

namespace dt {
namespace {

constexpr int kTraceThreads = 128;
constexpr int kBwdThreads = 128;

// minimum resident blocks per SM (register caps); tuned in profiles/r01_launch_bounds.txt
#ifndef DT_TRAV_MINB
#define DT_TRAV_MINB 1
#endif
#ifndef DT_SHADE_MINB
#define DT_SHADE_MINB 1
#endif
#ifndef DT_BWD_MINB
#define DT_BWD_MINB 1
#endif
#if DT_TRAV_MINB > 1
#define DT_TRAV_LB __launch_bounds__(kTraceThreads, DT_TRAV_MINB)
#else
#define DT_TRAV_LB __launch_bounds__(kTraceThreads)
#endif
// camera-ray kernel: 12 blocks / SM (r02 sweep, C3 trace0 ms: 8 / 9 / 10 / 12 blocks: 8.20 /
// 8.13 / 8.08 / 7.99; occupancy beats the spills of the float64 camera ray and env lookup)
#ifndef DT_PRIM_MINB
#define DT_PRIM_MINB 12
#endif
#ifndef DT_PRIM_VOL_MINB
#define DT_PRIM_VOL_MINB 8             // the volumetric-env variant (32-sample env integral) spills below 64
#endif
#define DT_PRIM_LB __launch_bounds__(kTraceThreads, VOL ? DT_PRIM_VOL_MINB : DT_PRIM_MINB)
#if DT_SHADE_MINB > 1
#define DT_SHADE_LB __launch_bounds__(kTraceThreads, DT_SHADE_MINB)
#else
#define DT_SHADE_LB __launch_bounds__(kTraceThreads)
#endif
#if DT_BWD_MINB > 1
#define DT_BWD_LB __launch_bounds__(kBwdThreads, DT_BWD_MINB)
#else
#define DT_BWD_LB __launch_bounds__(kBwdThreads)
#endif

// register caps of the sigma-grid kernels (k_*_grid: their cooperative walks inflate the
// allocation; measured: tools/sweep_regs.sh)
#ifndef DT_SHADE_GRID_REGS
#define DT_SHADE_GRID_REGS 80
#endif
#ifndef DT_BWD_GRID_REGS
#define DT_BWD_GRID_REGS 96
#endif
// the same for the hash texture (uncapped they take 158 / 168 registers: 12 warps per SM on
// a walk bound by the latency of its table fetches)
#ifndef DT_SHADE_HASH_REGS
#define DT_SHADE_HASH_REGS 128
#endif
#ifndef DT_BWD_HASH_REGS
#define DT_BWD_HASH_REGS 96
#endif

DT_D int fetch_work(int* counter, int chunk = 32) {
  int base = 0;
  if (lane_id() == 0) base = atomicAdd(counter, chunk);
  return __shfl_sync(~0u, base, 0);
}


// Hit-first lane order over a warp's window of 32 R records (R rounds of 32, R = DT_WIN_ROUNDS):
// records of class 0 (a traced hit: interface path) first, then class 1 (a miss: environment
// path), then class 2 (nothing to do).  The per-record code has two long, disjoint paths, so
// warps that mix them run both at half width; sorted, each round is (nearly) uniform.
// c[h]: class of window offset 32 h + lane; ord[h]: the offset this lane processes in round h.
// slot: the warp's 32 R bytes of shared memory.  R = 2 measured best (R = 4: C4 -0.8 %, C3 +1.6 %,
// C4H +1.5 % ms/step; R = 1: C3 +9.6 %; profiles/r02_traversal_sweep.txt).
#ifndef DT_WIN_ROUNDS
#define DT_WIN_ROUNDS 2
#endif
template <int R>
DT_D void hit_first_order_r(const int (&c)[R], unsigned char* slot, int (&ord)[R]) {
  const unsigned lt = lanemask_lt();
  unsigned b[3][R];
  int n[3] = {0, 0, 0};
#pragma unroll
  for (int h = 0; h < R; ++h)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      b[q][h] = __ballot_sync(~0u, c[h] == q);
      n[q] += __popc(b[q][h]);
    }
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int q = c[h];
    int r = q == 0 ? 0 : q == 1 ? n[0] : n[0] + n[1];
#pragma unroll
    for (int g = 0; g < R; ++g)
      if (g < h) r += __popc(q == 0 ? b[0][g] : q == 1 ? b[1][g] : b[2][g]);
    r += __popc((q == 0 ? b[0][h] : q == 1 ? b[1][h] : b[2][h]) & lt);
    DT_CHECK(r >= 0 && r < 32 * R);
    slot[r] = (unsigned char)(32 * h + lane_id());
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < R; ++h) ord[h] = slot[32 * h + lane_id()];
  __syncwarp();
}

// first record index of level k >= 1
DT_D int64_t level_base(const int* lvl, int k) {
  int64_t off = 0;
  for (int j = 1; j < k; ++j) off += lvl[LV_CNT + j];
  return off;
}

DT_D void sig_add(unsigned long long* sig, int64_t r, uint64_t key) {
  if (sig) atomicAdd(sig + r, (unsigned long long)dt_mix64(key));
}

// per-warp sum of the traversal counters, one 64-bit atomic per warp
DT_D void flush_counters(unsigned long long* c, int visits, int tests) {
  unsigned long long v = (unsigned long long)visits, t = (unsigned long long)tests;
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(~0u, v, o);
    t += __shfl_xor_sync(~0u, t, o);
  }
  if (lane_id() == 0 && c) {
    atomicAdd(c, v);
    atomicAdd(c + 1, t);
  }
}

// Shade one traced segment (record idx at level k) and spawn its children into level k+1.
// The traversal chose the face (float32 candidate search); the hit point, barycentrics,
// normals and the interface are recomputed here in float64 from the float64 ray state.
// All 32 lanes of the warp must call this (the compaction is a warp collective).
template <int ABS, bool VOL>
DT_D void shade_and_spawn(const FwdLaunch& a, double ior, int64_t child_off, int64_t lim, int k, int max_depth,
                          bool valid, int64_t idx, double3 o, double3 d, int64_t ray, uint32_t pos, float3 thr, float w,
                          int face, int i0, int i1, int i2) {
  const DevScene& s = a.s;
  bool is_hit = valid && face >= 0;
  bool spawn_r = false, spawn_t = false, need_tau = false, capped = false, volx = false;
  double3 x = d3(0, 0, 0), wr = x, wt = x;
  float3 tau = f3(1, 1, 1), capL = f3(0, 0, 0), Vx = capL;
  float Tx = 1.f;
  float R = 0.f, T = 0.f;
  if (valid) {
    if (!is_hit) {
      float Tm = 1.f;
      VolMom mom;
      float3 L = env_escape<VOL>(s, o, d, f3(0, 0, 0), nullptr, nullptr, &Tm, &mom);   // P:160 step 3 (R30)
      __stcs(a.r.hit + idx, make_float4(__int_as_float(-1), 0.f, 0.f, __int_as_float(RF_MISS)));
      __stcs(a.r.lsub + idx, f4(L, __int_as_float(-1)));
      __stcs(a.r.tau + idx, make_float4(Tm, Tm, Tm, __int_as_float(-1)));
      if (VOL) {                             // the volume's moments, for the backward
        __stcs(a.r.mq + idx, f4(mom.Qc, mom.odM));
        __stcs(a.r.mg + idx, f4(mom.Go, 0.f));
      }
      sig_add(a.sig_t, ray, topo_key(pos, EV_MISS));
      sig_add(a.sig_f, ray, face_key(pos, EV_MISS, -1));
    } else if (k == max_depth && s.cap_policy == 0 && !VOL) {
      // a hit at D_max under CAP_ZERO (R13, R34): the branch is discarded -- radiance and
      // gradient are zero whichever face or side was hit, so only "it hit" is recorded: no
      // vertex fetch, no interface, no interior transmittance (a sigma-grid walk at C4)
      capped = true;
      __stcs(a.r.hit + idx, make_float4(0.f, 0.f, 0.f, __int_as_float(RF_CAPPED)));
      sig_add(a.sig_t, ray, topo_key(pos, EV_CAP_DROP));
      sig_add(a.sig_f, ray, face_key(pos, EV_CAP_DROP, -1));
      if (a.capw) atomicAdd(a.capw + ray, w);
    } else {
      double3 v0, e1, e2;
      double t, u, v;
      tri64(s, i0, i1, i2, v0, e1, e2);
      mt64(o, d, v0, e1, e2, t, u, v);                                        // R15, float64
      const bool inside = dot(d, cross(e1, e2)) > 0.0;                        // R8
      x = o + d * t;
      need_tau = inside;
      volx = VOL && !inside;                                                  // exterior, volumetric env
      if (volx) {                                                             // R30
        VolMom mom;
        env_volume(s, f3(o), f3(x), Vx, Tx, &mom);
        __stcs(a.r.mq + idx, f4(mom.Qc, mom.odM));                            // for the backward
        __stcs(a.r.mg + idx, f4(mom.Go, 0.f));
      }
      if (k == max_depth) {                                                   // capped (R12, R13)
        capped = true;
        if (s.cap_policy == 1) capL = env_eval(s, o, d, f3(0, 0, 0), nullptr, nullptr);   // times tau below
        int fl = RF_CAPPED | (inside ? RF_INSIDE : 0);
        __stcs(a.r.hit + idx, make_float4(__int_as_float(i0), __int_as_float(i1), 0.f, __int_as_float(fl)));
        __stcs(a.r.thr + idx, f4(thr, __int_as_float(i2)));
        int ev = inside ? EV_CAP_IN : EV_CAP_OUT;
        sig_add(a.sig_t, ray, topo_key(pos, ev));
        sig_add(a.sig_f, ray, face_key(pos, ev, face));
        if (a.capw) atomicAdd(a.capw + ray, w);
      } else {
        Shade S;
        shade_forward(s, ior, i0, i1, i2, e1, e2, d, u, v, inside, S);
        R = (float)S.R;
        T = (float)S.T;
        wr = S.wr;
        wt = S.wt;
        spawn_r = true;                                                       // P:161 (R5)
        spawn_t = !S.tir;
        int fl = (inside ? RF_INSIDE : 0) | (S.tir ? RF_TIR : 0) | (S.degen ? RF_DEGEN : 0);
        __stcs(a.r.hit + idx, make_float4(__int_as_float(i0), __int_as_float(i1), R, __int_as_float(fl)));
        __stcs(a.r.thr + idx, f4(thr, __int_as_float(i2)));
        int ev = inside ? (S.tir ? EV_HIT_IN_TIR : EV_HIT_IN) : (S.tir ? EV_HIT_OUT_TIR : EV_HIT_OUT);
        sig_add(a.sig_t, ray, topo_key(pos, ev));
        sig_add(a.sig_f, ray, face_key(pos, ev, face));
      }
    }
  }
  // interior transmittance of the segment o -> x (R9)
  if (ABS == 0) {
    if (need_tau) tau = transmittance_const(s, o, x);
  } else {
    const GridMap gm = grid_map(s);
    const float3 of = f3(o), xf = f3(x);
    for (unsigned m = __ballot_sync(~0u, need_tau); m;) {                // cooperative walks
      int myq;
      constexpr int G = WalkLanes<ABS>::fwd;
      const int src = group_take<G>(m, myq), sl = max(src, 0);
      const float3 Sd = group_optical_depth<G, ABS>(s, gm, shfl3(of, sl), shfl3(xf, sl), src >= 0);
      const float3 mine = shfl3(Sd, max(myq, 0) * G);
      if (myq >= 0) tau = f3(expf(-mine.x), expf(-mine.y), expf(-mine.z));
    }
  }
  if (volx) tau = f3(Tx, Tx, Tx);            // exterior: the continuation is seen through the env volume
  if (capped) {
    __stcs(a.r.lsub + idx, f4(volx ? Vx + capL * tau : capL * tau, __int_as_float(-1)));
    __stcs(a.r.tau + idx, f4(tau, __int_as_float(-1)));
  }
  // warp-ballot compaction of the children: the warp's reflect children first, then its
  // refract children, each group contiguous in level k+1
  unsigned mr = __ballot_sync(~0u, spawn_r), mt = __ballot_sync(~0u, spawn_t);
  int nr = __popc(mr), nt = __popc(mt);
  int base = 0;
  if (nr + nt > 0) {
    if (lane_id() == 0) base = atomicAdd(a.lvl + LV_CNT + k + 1, nr + nt);
    base = __shfl_sync(~0u, base, 0);
  }
  if (spawn_r) {
    const int64_t off = child_off;
    int64_t cr = -1, ct = -1;
    int64_t j = off + base + __popc(mr & lanemask_lt());
    if (j < lim) {
      cr = j;
      stcs64(a.r.o + j, mk64(x, (int)ray, 0u));
      stcs64(a.r.d + j, mk64(wr, 0, pos * 2u));
      __stcs(a.r.thr + j, f4(thr * tau * R, w * R));
    } else {
      a.lvl[LV_OVERFLOW] = 1;
    }
    if (spawn_t) {
      j = off + base + nr + __popc(mt & lanemask_lt());
      if (j < lim) {
        ct = j;
        stcs64(a.r.o + j, mk64(x, (int)ray, 0u));
        stcs64(a.r.d + j, mk64(wt, 0, pos * 2u + 1u));
        __stcs(a.r.thr + j, f4(thr * tau * T, w * T));
      } else {
        a.lvl[LV_OVERFLOW] = 1;
      }
    }
    __stcs(a.r.tau + idx, f4(tau, __int_as_float((int)ct)));
    __stcs(a.r.lsub + idx, f4(Vx, __int_as_float((int)cr)));            // V: the segment's own env emission
  }
}

// Level 0: camera rays.  Each warp takes 32 pixels of an 8x4 tile (or 32 consecutive
// entries of the caller's pixel list), culls against the root box, traverses (float32
// candidate search with the rounded ray), and records only the hitting rays, with their
// float64 ray state (misses write their env radiance straight to rgb).
template <bool VOL>
__global__ void DT_PRIM_LB k_trace_primary(FwdLaunch a, int max_depth) {
  __shared__ int sstack[kStackShared * kTraceThreads];
  const DevScene& s = a.s;
  float3 blo = f3(s.scal[0], s.scal[1], s.scal[2]), bhi = f3(s.scal[3], s.scal[4], s.scal[5]);
  int err = 0, visits = 0, tests = 0, traced = 0;
  int base = fetch_work(a.lvl + LV_WORK_PRIMARY);
  while (base < a.n_items) {
    int next = 0;                     // the next chunk's atomic is in flight during this one
    if (lane_id() == 0) next = atomicAdd(a.lvl + LV_WORK_PRIMARY, 32);
    int64_t item = (int64_t)base + lane_id();
    bool valid = item < a.n_items;
    int64_t pid = 0;
    if (valid) {
      if (a.pids) {
        pid = a.pids[item];
      } else if (a.shard_tile > 0) {   // tile shard: slot item / T^2, 8x4 micro-tiles inside the tile
        const int T = a.shard_tile, T2 = T * T;
        const int64_t slot = item / T2;
        const int w = (int)(item - slot * T2);
        const int64_t tid = a.tile_ids ? (int64_t)a.tile_ids[slot] : a.shard_rank + slot * a.shard_count;
        const int view = (int)(tid / a.stiles_per_view);
        const int tv = (int)(tid - (int64_t)view * a.stiles_per_view);
        const int ty = tv / a.stiles_x, tx = tv - ty * a.stiles_x;
        const int mt = w >> 5, l = w & 31, mpr = T >> 3;
        const int px = tx * T + (mt % mpr) * 8 + (l & 7), py = ty * T + (mt / mpr) * 4 + (l >> 3);
        DT_CHECK(view >= 0 && view < a.n_views && px < a.W && py < a.H);
        pid = ((int64_t)view * a.H + py) * a.W + px;
      } else {
        int64_t tile = item >> 5;
        int l = (int)(item & 31);
        int view = (int)(tile / a.tiles_per_view);
        int tv = (int)(tile - (int64_t)view * a.tiles_per_view);
        int ty = tv / a.tiles_x, tx = tv - ty * a.tiles_x;
        int px = tx * 8 + (l & 7), py = ty * 4 + (l >> 3);
        valid = px < a.W && py < a.H;
        pid = ((int64_t)view * a.H + py) * a.W + px;
      }
    }
    int64_t ray = a.pids || a.shard_tile > 0 ? item : pid;
    double3 o64 = d3(0, 0, 0), d64 = d3(0, 0, 1);
    int face = -1;
    float t = 0.f, u = 0.f, v = 0.f;
    bool inbox = false;
    if (valid) {
      camera_ray64(a.K, a.c2w, a.W, a.H, pid, o64, d64);
      float tn;
      inbox = slab(blo.x, bhi.x, blo.y, bhi.y, blo.z, bhi.z, f3(o64), safe_inv(f3(d64)), kInf, tn);
      traced += inbox;
      if (inbox && a.segc) a.segc[ray] += 1;          // one lane per ray: no atomic needed
    }
    if (inbox) face = traverse(s, f3(o64), f3(d64), 0.0f, t, u, v, sstack + threadIdx.x, kTraceThreads, err, visits, tests);
    if (valid) {
      if (face < 0) {
        float3 L = env_escape<VOL>(s, o64, d64, f3(0, 0, 0), nullptr, nullptr);
        a.rgb[3 * ray] = L.x; a.rgb[3 * ray + 1] = L.y; a.rgb[3 * ray + 2] = L.z;
        sig_add(a.sig_t, ray, topo_key(1u, EV_MISS));
        sig_add(a.sig_f, ray, face_key(1u, EV_MISS, -1));
      }
    }
    bool rec = valid && face >= 0;
    unsigned m = __ballot_sync(~0u, rec);
    int rb = 0;
    if (m) {
      if (lane_id() == 0) rb = atomicAdd(a.lvl + LV_CNT + 0, __popc(m));
      rb = __shfl_sync(~0u, rb, 0);
    }
    int64_t idx = a.cap - 1 - (rb + __popc(m & lanemask_lt()));
    if (rec && idx < 0) { a.lvl[LV_OVERFLOW] = 1; rec = false; }
    if (rec) {
      stcs64(a.r.o + idx, mk64(o64, (int)ray, 0u));
      stcs64(a.r.d + idx, mk64(d64, 0, 1u));
      __stcs(a.r.thr + idx, make_float4(1.f, 1.f, 1.f, 1.f));
      __stcs(a.r.hit + idx, hit_record(s, face));   // shaded by k_shade_level(0)
    }
    base = __shfl_sync(~0u, next, 0);
  }
  if (err) a.lvl[LV_STACKERR] = 1;
  for (int o = 16; o > 0; o >>= 1) traced += __shfl_xor_sync(~0u, traced, o);
  if (lane_id() == 0 && traced) atomicAdd(a.lvl + LV_TRACED, traced);
  flush_counters(a.counters + 2, visits, tests);   // primary rays: counters [2], [3]
}

// Shading of level k (K10): reads each record's ray and traversal result, evaluates the
// event and spawns the children into level k+1 (warp-ballot compaction).  Level 0 needs
// the final level-0 count, so it always runs after the traversal pass.
// Each warp takes a window of 64 records and shades them in two rounds of 32 in hit-first
// lane order (hit_first_order_r).  Work distribution: warps take 64-record windows from the
// level's counter, the next window's atomic in flight while the current one is shaded -- a
// window's cost varies with its hit / miss mix (and with the interior walks of a sigma grid,
// a hash texture or a volumetric env), so a static stride left a tail (r02: constant-sigma C3
// shade 9.45 -> 8.92 ms; DT_SHADE_DYN=0 restores the static stride).
template <int ABS, bool VOL>
DT_D void shade_level_body(const FwdLaunch& a, int k, int max_depth) {
  if (a.lvl[LV_OVERFLOW]) return;   // arena too small: the host grows it and re-runs
  const double ior = a.s.ior_ptr ? (double)__ldg(a.s.ior_ptr) : (double)a.s.ior;
  // level offsets are fixed while this kernel runs (only level k+1's count grows): read once
  const int n = a.lvl[LV_CNT + k];
  const int64_t off = k == 0 ? 0 : level_base(a.lvl, k);
  const int64_t child_off = level_base(a.lvl, k + 1);
  const int64_t lim = a.cap - a.lvl[LV_CNT + 0];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#ifndef DT_SHADE_DYN
#define DT_SHADE_DYN 1
#endif
  constexpr bool kDyn = ABS != 0 || VOL || DT_SHADE_DYN;
  int* const ctr = a.lvl + LV_WORK_SHADE + k;
  constexpr int RW = DT_WIN_ROUNDS, WIN = 32 * RW;
  __shared__ unsigned char sslot[kTraceThreads * RW];
  int64_t wbase = kDyn ? (int64_t)fetch_work(ctr, WIN) : (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * RW;
  int round = 0, next = 0;
  int ord[RW];
  while (wbase < n) {
    if (round == 0 && kDyn && lane_id() == 0) next = atomicAdd(ctr, WIN);
    if (round == 0) {
      int c[RW];
#pragma unroll
      for (int h = 0; h < RW; ++h) {
        const int64_t it = wbase + 32 * h + lane_id();
        c[h] = 2;
        if (it < n) c[h] = __float_as_int(a.r.hit[k == 0 ? a.cap - 1 - it : off + it].x) >= 0 ? 0 : 1;
      }
      hit_first_order_r<RW>(c, sslot + RW * (threadIdx.x & ~31), ord);
    }
    int my = ord[0];
#pragma unroll
    for (int h = 1; h < RW; ++h)
      if (round == h) my = ord[h];
    const int64_t item = wbase + my;
    const bool valid = item < n;
    const int64_t idx = k == 0 ? a.cap - 1 - item : off + item;
    double3 o = d3(0, 0, 0), d = d3(0, 0, 1);
    float3 thr = f3(0, 0, 0);
    float w = 0.f;
    int64_t ray = 0;
    uint32_t pos = 0;
    int face = -1, i0 = 0, i1 = 0, i2 = 0;
    if (valid) {
      DT_CHECK(idx >= 0 && idx < a.cap);
      const Vec64 ro = ldcs64(a.r.o + idx), rd = ldcs64(a.r.d + idx);
      const float4 rt = __ldcs(a.r.thr + idx), h = __ldcs(a.r.hit + idx);
      o = xyz(ro); d = xyz(rd); thr = f3(rt); w = rt.w;
      ray = ro.i;
      pos = rd.u;
      face = __float_as_int(h.x);
      i0 = __float_as_int(h.y); i1 = __float_as_int(h.z); i2 = __float_as_int(h.w);
    }
    if (valid && k > 0 && a.segc) atomicAdd(a.segc + ray, 1);
    shade_and_spawn<ABS, VOL>(a, ior, child_off, lim, k, max_depth, valid, idx, o, d, ray, pos, thr, w, face, i0, i1,
                              i2);
    if (++round == RW) {
      round = 0;
      wbase = kDyn ? (int64_t)__shfl_sync(~0u, next, 0) : wbase + RW * stride;
    }
  }
}

template <int ABS, bool VOL>
__global__ void DT_SHADE_LB k_shade_level(FwdLaunch a, int k, int max_depth) {
  shade_level_body<ABS, VOL>(a, k, max_depth);
}
template <bool VOL>
__global__ void __maxnreg__(DT_SHADE_GRID_REGS)
    k_shade_level_grid(FwdLaunch a, int k, int max_depth) {
  shade_level_body<1, VOL>(a, k, max_depth);
}
template <bool VOL>
__global__ void __maxnreg__(DT_SHADE_HASH_REGS)
    k_shade_level_hash(FwdLaunch a, int k, int max_depth) {
  shade_level_body<2, VOL>(a, k, max_depth);
}
#ifndef DT_SHADE_VOL_REGS
#define DT_SHADE_VOL_REGS 96
#endif
__global__ void __maxnreg__(DT_SHADE_VOL_REGS) k_shade_level_vol(FwdLaunch a, int k, int max_depth) {
  shade_level_body<0, true>(a, k, max_depth);
}

// Traversal of level k >= 1 (K9): closest hit only, hit = (face, t, u, v) written back into
// the record (the float32 candidate search; shade recomputes the hit in float64).  Lanes that
// finish their ray refill from the level's queue (one warp-aggregated atomic per refill), so
// short reflected rays do not idle a warp behind long refracted ones.
constexpr int kStepBudget = 16;   // traversal steps between refill votes (swept: 8 / 16 / 32)
__global__ void DT_TRAV_LB k_traverse_level(FwdLaunch a, int k) {
  __shared__ int sstack_all[kStackShared * kTraceThreads];
  const DevScene& s = a.s;
  if (a.lvl[LV_OVERFLOW]) return;
  const float t_lo = a.t_eps * s.scal[6];                                      // R17
  const int n = a.lvl[LV_CNT + k];
  const int64_t off = level_base(a.lvl, k);
  int* work = a.lvl + LV_WORK_TRACE + k;
  int* sstack = sstack_all + threadIdx.x;
  int lstack[kStackLocal];
  int err = 0, visits = 0, tests = 0;
  int item = -1;                       // -1: needs a ray; >= n: queue exhausted
  int pend = -1;                       // finished ray whose hit record is stored next round
  float4 ph = make_float4(0.f, 0.f, 0.f, 0.f);
  float3 o = f3(0, 0, 0), d = f3(0, 0, 1), inv = f3(0, 0, 0);
  Trav T;
  trav_init(T);
  while (true) {
    unsigned need = __ballot_sync(~0u, item < 0);
    if (need) {                        // one warp-aggregated atomic on the level's queue
      const int leader = __ffs(need) - 1;
      int base = 0;
      if (lane_id() == leader) base = atomicAdd(work, __popc(need));
      base = __shfl_sync(~0u, base, leader);
      if (item < 0) {
        const int j = base + __popc(need & lanemask_lt());
        if (j < n) {
          item = j;
          DT_CHECK(off + j < a.cap);
          o = f3(xyz(ldcs64(a.r.o + off + j)));       // the float64 ray, rounded for the search
          d = f3(xyz(ldcs64(a.r.d + off + j)));
          inv = safe_inv(d);
          trav_init(T);
        } else {
          item = n;
        }
      }
    }
    if (__all_sync(~0u, item >= n)) break;
    bool done = false;
    if (item >= 0 && item < n) {
      for (int step = 0; step < kStepBudget && !done; ++step)
        done = trav_step(s, o, d, inv, t_lo, T, sstack, kTraceThreads, lstack, err, visits, tests);
    }
    // the hit record of a ray finished one round earlier: its face's vertex indices were
    // fetched then and have arrived during this round's steps
    if (pend >= 0) {
      __stcs(a.r.hit + off + pend, ph);
      pend = -1;
    }
    if (done) {
      ph = hit_record(s, T.best);
      pend = item;
      item = -1;
    }
  }
  if (pend >= 0) __stcs(a.r.hit + off + pend, ph);
  if (err) a.lvl[LV_STACKERR] = 1;
  flush_counters(a.counters, visits, tests);
}

// Bottom-up radiance: L = tau * (R L_r + T L_t); level 0 writes the pixel.
__global__ void k_gather(FwdLaunch a, int k) {
  if (a.lvl[LV_OVERFLOW]) return;
#ifdef DT_CHECK_SELFTEST
  DT_CHECK(false);                     // tools/checked_build.sh: the check plumbing reports a failure
#endif
  const int n = a.lvl[LV_CNT + k];
  const int64_t off = k == 0 ? 0 : level_base(a.lvl, k);
  for (int64_t item = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; item < n; item += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = k == 0 ? a.cap - 1 - item : off + item;
    DT_CHECK(idx >= 0 && idx < a.cap);
    float4 h = a.r.hit[idx];
    int fl = __float_as_int(h.w);
    float4 ls = a.r.lsub[idx];
    float3 L;
    if (fl & (RF_MISS | RF_CAPPED)) {
      L = f3(ls);
    } else {
      float4 tu = a.r.tau[idx];
      int cr = __float_as_int(ls.w), ct = __float_as_int(tu.w);
      float R = h.z;
      DT_CHECK(cr < a.cap && ct < a.cap);
      float3 Lr = cr >= 0 ? f3(a.r.lsub[cr]) : f3(0, 0, 0);
      float3 Lt = ct >= 0 ? f3(a.r.lsub[ct]) : f3(0, 0, 0);
      L = f3(ls) + f3(tu) * (Lr * R + Lt * (1.0f - R));   // own emission (R30; 0 otherwise) + tau * children
      a.r.lsub[idx] = f4(L, ls.w);
    }
    if (k == 0) {
      int64_t ray = a.r.o[idx].i;
      a.rgb[3 * ray] = L.x; a.rgb[3 * ray + 1] = L.y; a.rgb[3 * ray + 2] = L.z;
    }
  }
}

// ----------------------------------------------------------------------------- backward
DT_D void atomic_add3(float4* p, float3 v) {
  atomicAdd(p, make_float4(v.x, v.y, v.z, 0.0f));
}

// Backward replay of level k (K12): per record, the local VJP at fixed topology, evaluated at
// the float64 ray state the forward used: the hit and the interface state are recomputed in
// float64 exactly as the forward did, then rounded to float32 for the Jacobian-times-adjoint
// arithmetic (the adjoints are float32; no state error propagates along the path).  Three
// phases per warp-iteration so that the sigma-grid walks (ABS = grid) run warp-cooperatively:
// (A) per lane: env / interface adjoints up to the interior segment's optical-depth adjoint
// gS; (B) the transmittance adjoints of the warp's interior segments, one segment at a time
// by the whole warp (or per lane for constant sigma); (C) per lane: x = o + t d and the
// Moller-Trumbore reverse, vertex and normal atomics, parent-slot adjoints.
// Each warp takes a window of 64 records in two rounds of 32, interface records first.
template <int ABS, bool VOL>
DT_D void backward_level_body(const BwdLaunch& a, int k, int max_depth, int64_t cap) {
  const DevScene& s = a.s;
  if (a.lvl[LV_OVERFLOW]) return;   // an overflowed (asynchronous) forward: nothing valid to replay
  const double ior = s.ior_ptr ? (double)__ldg(s.ior_ptr) : (double)s.ior;
  const int n = a.lvl[LV_CNT + k];
  const int64_t off = k == 0 ? 0 : level_base(a.lvl, k);
  float gior = 0.0f;
  float3 gsc = f3(0, 0, 0);
  int vsamp = 0;                       // volumetric-env samples replayed (the bench's roofline)
  constexpr int RW = DT_WIN_ROUNDS, WIN = 32 * RW;
  __shared__ unsigned char sslot[kBwdThreads * RW];
  // 64-record windows taken from the level's counter (the next window's atomic in flight while
  // this one is replayed): window costs vary with the hit / miss mix, so a static stride leaves
  // a tail
  int* const ctr = a.lvl + LV_WORK_BWD + k;
  int64_t wb = fetch_work(ctr, WIN);
  int nx = 0;
  if (lane_id() == 0) nx = atomicAdd(ctr, WIN);
  while (wb < n) {
  int ord[RW];
  {
    int c[RW];
#pragma unroll
    for (int h = 0; h < RW; ++h) {
      const int64_t it = wb + 32 * h + lane_id();
      c[h] = 2;
      if (it < n) {
        const int f = __float_as_int(a.r.hit[k == 0 ? cap - 1 - it : off + it].w);
        c[h] = (f & RF_MISS) ? 1 : ((f & RF_CAPPED) && s.cap_policy == 0 && !VOL) ? 2 : 0;
      }
    }
    hit_first_order_r<RW>(c, sslot + RW * (threadIdx.x & ~31), ord);
  }
#pragma unroll 1
  for (int round = 0; round < RW; ++round) {
    int my = ord[0];
#pragma unroll
    for (int h = 1; h < RW; ++h)
      if (round == h) my = ord[h];
    const int64_t item = wb + my;
    const bool valid = item < n;
    int64_t idx = 0;
    float3 go = f3(0, 0, 0), gd = go, gx = go, gS = go, gNk[3];
    float3 of = go, xf = go, df = go, dhf = go, e1f = go, e2f = go;   // float32 copies for the reverse
    float t = 0.f, u = 0.f, v = 0.f, gu = 0.f, gv = 0.f, idet = 0.f, lch = 0.f;
    int fl = 0, i0 = 0, i1 = 0, i2 = 0;
    bool geo = false, walk = false;
    // ---- (A)
    if (valid) {
      idx = k == 0 ? cap - 1 - item : off + item;
      DT_CHECK(idx >= 0 && idx < cap);
      const Vec64 ro = ldcs64(a.r.o + idx), rd = ldcs64(a.r.d + idx);
      const float4 rt = a.r.thr[idx], h = a.r.hit[idx];
      const double3 o = xyz(ro), d = xyz(rd);
      const int64_t ray = ro.i;
      fl = __float_as_int(h.w);
      const float* g = a.grad_rgb + 3 * ray;
      const float3 adj = f3(__ldg(g), __ldg(g + 1), __ldg(g + 2)) * f3(rt);   // a_n = grad * throughput
      const bool volx = VOL && !(fl & (RF_MISS | RF_INSIDE));                 // exterior segment, R30
      VolMom mom;
      if (VOL && !(fl & RF_INSIDE)) {                                         // recorded by the forward
        const float4 q = a.r.mq[idx], g4 = a.r.mg[idx];
        mom.Qc = f3(q);
        mom.odM = q.w;
        mom.Go = f3(g4);
      }
      if (fl & RF_MISS) {
        float Tm = a.r.tau[idx].x;
        env_escape<VOL>(s, o, d, adj, &go, &gd, &Tm, &mom);
        if (VOL) vsamp += s.env_nsamp;
      } else if ((fl & RF_CAPPED) && s.cap_policy == 0 && !volx) {
        // capped branches return 0: no dependence
      } else {
        geo = true;
        i0 = __float_as_int(h.x); i1 = __float_as_int(h.y); i2 = __float_as_int(rt.w);   // from the shade
        const bool inside = (fl & RF_INSIDE) != 0;
        double3 v0, e1, e2;
        double t64, u64, v64;
        tri64(s, i0, i1, i2, v0, e1, e2);
        idet = (float)mt64(o, d, v0, e1, e2, t64, u64, v64);                 // the forward's hit, replayed
        const double3 x = o + d * t64;
        of = f3(o); xf = f3(x); df = f3(d); e1f = f3(e1); e2f = f3(e2);
        t = (float)t64; u = (float)u64; v = (float)v64;
        lch = (float)length(x - o);
        dhf = f3(d * rsqrt64(dot(d, d)));
        const float4 tu = a.r.tau[idx];
        const float3 tau = f3(tu);
        if (fl & RF_CAPPED) {                                                 // CAP_ENV leaf
          if (volx) {                                                         // V + Tn * (E or 0)
            float aT = 0.f;
            if (s.cap_policy == 1) aT = dot(adj, env_eval(s, o, d, adj * tau, &go, &gd));
            env_volume_bwd(s, of, xf, adj, aT, tau.x, mom, go, gx);
            vsamp += s.env_nsamp;
          } else {
            const float3 E = env_eval(s, o, d, adj * tau, &go, &gd);
            if (inside) { walk = true; gS = -(adj * E * tau); }
          }
          gNk[0] = gNk[1] = gNk[2] = f3(0, 0, 0);
        } else {
          ShadeF S;
          {
            Shade S64;
            shade_forward(s, ior, i0, i1, i2, e1, e2, d, u64, v64, inside, S64);
            S = shade_f32(S64);
          }
          const float4 ls = a.r.lsub[idx];
          const int cr = __float_as_int(ls.w), ct = __float_as_int(tu.w);
          DT_CHECK(cr < cap && ct < cap && (cr < 0 || cr > idx - (k == 0 ? cap : 0)));
          float3 Lr = f3(0, 0, 0), Lt = f3(0, 0, 0);
          float3 gwr = f3(0, 0, 0), gwt = f3(0, 0, 0);
          if (cr >= 0) { Lr = f3(a.r.lsub[cr]); gx += f3(a.r.go[cr]); gwr = f3(a.r.gd[cr]); }
          if (ct >= 0) { Lt = f3(a.r.lsub[ct]); gx += f3(a.r.go[ct]); gwt = f3(a.r.gd[ct]); }
          const float3 ap = adj * tau;
          const float Rf = h.z;                                               // R, as the forward stored it
          const float3 Lc = Lr * Rf + Lt * (1.0f - Rf);
          const float gR = S.tir ? 0.0f : dot(ap, Lr - Lt);
          if (inside) { walk = true; gS = -(adj * Lc * tau); }
          if (volx) {                                                         // V + Tn * Lc (R30)
            env_volume_bwd(s, of, xf, adj, dot(adj, Lc), tau.x, mom, go, gx);
            vsamp += s.env_nsamp;
          }
          float3 gd_s;
          float gi;
          const float3 n0 = f3(xyz(ldg_d4(s.nrm + i0))), n1 = f3(xyz(ldg_d4(s.nrm + i1))),
                       n2 = f3(xyz(ldg_d4(s.nrm + i2)));
          shade_backward(S, df, gR, gwr, gwt, n0, n1, n2, gd_s, gu, gv, gNk, gi);
          gd += gd_s;
          gior += gi;
        }
      }
    }
    // ---- (B) interior transmittance o -> x
    if (ABS == 0) {
      if (walk) transmittance_const_backward(s, lch, dhf, gS, gx, go, gsc);
    } else {
      const GridMap gm = grid_map(s);
      for (unsigned m = __ballot_sync(~0u, walk); m;) {
        int myq;
        constexpr int G = WalkLanes<ABS>::bwd;
        const int src = group_take<G>(m, myq), sl = max(src, 0);
        float3 wgx, wgo;
        group_transmittance_backward<G, ABS>(s, gm, shfl3(of, sl), shfl3(xf, sl), shfl3(gS, sl), src >= 0, a.dsig, wgx,
                                             wgo);
        const float3 mx = shfl3(wgx, max(myq, 0) * G), mo = shfl3(wgo, max(myq, 0) * G);
        if (myq >= 0) { gx += mx; go += mo; }
      }
    }
    // ---- (C) x = o + t d, then the Moller-Trumbore solve
    if (geo) {
      go += gx;
      gd += gx * t;
      float3 gVk[3];
      mt_backward(df, e1f, e2f, idet, t, u, v, gu, gv, dot(gx, df), go, gd, gVk);
      atomic_add3(a.dV + i0, gVk[0]);
      atomic_add3(a.dV + i1, gVk[1]);
      atomic_add3(a.dV + i2, gVk[2]);
      if (!(fl & RF_CAPPED)) {
        atomic_add3(a.dN + i0, gNk[0]);
        atomic_add3(a.dN + i1, gNk[1]);
        atomic_add3(a.dN + i2, gNk[2]);
      }
    }
    if (valid && k > 0) {                                                     // camera rays: dropped (R22)
      a.r.go[idx] = f4(go, 0.f);
      a.r.gd[idx] = f4(gd, 0.f);
    }
  }
  wb = __shfl_sync(~0u, nx, 0);
  if (lane_id() == 0) nx = atomicAdd(ctr, WIN);
  }
  // warp reductions of the scalar adjoints
  for (int o = 16; o > 0; o >>= 1) {
    gior += __shfl_xor_sync(~0u, gior, o);
    gsc.x += __shfl_xor_sync(~0u, gsc.x, o);
    gsc.y += __shfl_xor_sync(~0u, gsc.y, o);
    gsc.z += __shfl_xor_sync(~0u, gsc.z, o);
  }
  if (VOL) flush_walk_count(s.wcount ? s.wcount + 2 : nullptr, vsamp);
  if (lane_id() == 0) {
    if (gior != 0.0f) atomicAdd(a.dior, gior);
    if (ABS == 0 && (gsc.x != 0.0f || gsc.y != 0.0f || gsc.z != 0.0f)) {
      atomicAdd(a.dsig, make_float4(gsc.x, gsc.y, gsc.z, 0.f));
    }
  }
}

template <int ABS, bool VOL>
__global__ void DT_BWD_LB k_backward_level(BwdLaunch a, int k, int max_depth, int64_t cap) {
  backward_level_body<ABS, VOL>(a, k, max_depth, cap);
}
template <bool VOL>
__global__ void __maxnreg__(DT_BWD_GRID_REGS)
    k_backward_level_grid(BwdLaunch a, int k, int max_depth, int64_t cap) {
  backward_level_body<1, VOL>(a, k, max_depth, cap);
}
template <bool VOL>
__global__ void __maxnreg__(DT_BWD_HASH_REGS)
    k_backward_level_hash(BwdLaunch a, int k, int max_depth, int64_t cap) {
  backward_level_body<2, VOL>(a, k, max_depth, cap);
}
// constant sigma, shell env: latency bound (dependent record -> child / vertex / gradient
// fetches), so a register cap that buys occupancy pays (tools/sweep_regs.sh)
#ifndef DT_BWD_CONST_REGS
#define DT_BWD_CONST_REGS 88
#endif
__global__ void __maxnreg__(DT_BWD_CONST_REGS) k_backward_level_const(BwdLaunch a, int k, int max_depth, int64_t cap) {
  backward_level_body<0, false>(a, k, max_depth, cap);
}
// constant sigma, volumetric env: the per-sample texel Jacobians otherwise take 168 registers
#ifndef DT_BWD_VOL_REGS
#define DT_BWD_VOL_REGS 128
#endif
__global__ void __maxnreg__(DT_BWD_VOL_REGS) k_backward_level_vol(BwdLaunch a, int k, int max_depth, int64_t cap) {
  backward_level_body<0, true>(a, k, max_depth, cap);
}

// Vertex-normal chain (reverse of P:170-173): dN -> d(sum of unit face normals) per vertex,
// -> per face d/de1, d/de2 -> gathered back per vertex through the corner CSR.
__global__ void k_vn_bwd_vertex(const float4* __restrict__ dN, const D4* __restrict__ nrm, int nv, float4* __restrict__ gS) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const D4 n = nrm[v];
    const double3 g = d3(dN[v]), nn = xyz(n);
    gS[v] = n.w > 0.0 ? f4(f3((g - nn * dot(nn, g)) * (1.0 / n.w)), 0.f) : make_float4(0, 0, 0, 0);
  }
}

__global__ void k_vn_bwd_face(const float4* __restrict__ V, const int* __restrict__ F, const D4* __restrict__ fn,
                              const float4* __restrict__ gS, int nf, float4* __restrict__ fe) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x) {
    const D4 h4 = fn[f];
    if (!(h4.w > 0.0)) { fe[2 * f] = make_float4(0, 0, 0, 0); fe[2 * f + 1] = make_float4(0, 0, 0, 0); continue; }
    int i0 = F[3 * f], i1 = F[3 * f + 1], i2 = F[3 * f + 2];
    const double3 gh = d3(gS[i0]) + d3(gS[i1]) + d3(gS[i2]);
    const double3 h = xyz(h4);
    const double3 gc = (gh - h * dot(h, gh)) * (1.0 / h4.w);
    const double3 a = d3(V[i0]);
    const double3 e1 = d3(V[i1]) - a, e2 = d3(V[i2]) - a;
    fe[2 * f] = f4(f3(cross(e2, gc)), 0.f);      // d/de1 of c = e1 x e2
    fe[2 * f + 1] = f4(f3(cross(gc, e1)), 0.f);  // d/de2
  }
}

__global__ void k_vn_bwd_gather(const int* __restrict__ vstart, const unsigned* __restrict__ corner,
                                const float4* __restrict__ fe, int nv, float4* __restrict__ gVn) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    float3 acc = f3(0, 0, 0);
    for (int j = vstart[v]; j < vstart[v + 1]; ++j) {
      unsigned c = corner[j];
      unsigned f = c / 3, kk = c - 3 * f;
      float3 g1 = f3(fe[2 * f]), g2 = f3(fe[2 * f + 1]);
      acc += kk == 0 ? -(g1 + g2) : (kk == 1 ? g1 : g2);
    }
    gVn[v] = f4(acc, 0.f);
  }
}

__global__ void k_finalize(const float4* __restrict__ gV, const float4* __restrict__ gVn, int nv, float* __restrict__ out,
                           int acc) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    float3 g = f3(gV[v]) + f3(gVn[v]);
    if (acc) { out[3 * v] += g.x; out[3 * v + 1] += g.y; out[3 * v + 2] += g.z; }
    else { out[3 * v] = g.x; out[3 * v + 1] = g.y; out[3 * v + 2] = g.z; }
  }
}

// sigma [n][3] -> x-pairs: out[2i], out[2i+1] = (sigma_i, sigma_{i+1 along x}, 0, 0), 32 B per
// node so that one 256-bit load fetches both x-corners of a cell edge (res = x extent; the
// last x node of a row pairs with zeros; constant sigma: res = 1).
__global__ void k_pack_sigma(const float* __restrict__ in, float4* __restrict__ out, int64_t n, int res, int pairs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!pairs) {                     // plain float4 per node / table entry
      out[i] = make_float4(in[3 * i], in[3 * i + 1], in[3 * i + 2], 0.f);
      continue;
    }
    const bool nx = (i % res) + 1 < res;
    const float a = in[3 * i], b = in[3 * i + 1], c = in[3 * i + 2];
    const float d = nx ? in[3 * i + 3] : 0.f, e = nx ? in[3 * i + 4] : 0.f, f = nx ? in[3 * i + 5] : 0.f;
    out[2 * i] = make_float4(a, b, c, d);
    out[2 * i + 1] = make_float4(e, f, 0.f, 0.f);
  }
}

__global__ void k_unpack_add(const float4* __restrict__ src, float* __restrict__ dst, int64_t n, int acc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float4 g = src[i];
    if (acc) { dst[3 * i] += g.x; dst[3 * i + 1] += g.y; dst[3 * i + 2] += g.z; }
    else { dst[3 * i] = g.x; dst[3 * i + 1] = g.y; dst[3 * i + 2] = g.z; }
  }
}

__global__ void k_copy_add(const float* __restrict__ src, float* __restrict__ dst, int64_t n, int acc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = acc ? dst[i] + src[i] : src[i];
}

// L_color and its gradient, fused
__global__ void k_loss_color(const float* __restrict__ rgb, const float* __restrict__ tgt, int64_t n, float inv_b,
                             float* __restrict__ grad, float* __restrict__ loss) {
  float acc = 0.0f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n; i += (int64_t)gridDim.x * blockDim.x) {
    float c = tgt[i], e = rgb[i] - c;
    float we = e * c;
    acc += we * we;
    grad[i] = 2.0f * we * c * inv_b;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
  if (lane_id() == 0) atomicAdd(loss, acc * inv_b);
}

__global__ void k_count_segments(const int* __restrict__ lvl, int D, unsigned long long* __restrict__ seg) {
  if (lvl[LV_OVERFLOW]) return;
  unsigned long long s = (unsigned)lvl[LV_TRACED];
  for (int k = 1; k <= D; ++k) s += (unsigned)lvl[LV_CNT + k];
  *seg += s;
}

__global__ void k_normals_to_f32(const D4* __restrict__ nrm, int nv, float* __restrict__ out) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const D4 n = nrm[v];
    out[3 * v] = (float)n.x; out[3 * v + 1] = (float)n.y; out[3 * v + 2] = (float)n.z;
  }
}

__global__ void k_check_finite(const float* __restrict__ x, int64_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) *flag = 1;
}

__global__ void __launch_bounds__(kTraceThreads) k_debug_hit(DevScene s, const float* __restrict__ rays, int64_t n,
                                                             float t_lo, int brute, int* __restrict__ face,
                                                             float* __restrict__ tuv, int* err_flag) {
  __shared__ int sstack[kStackShared * kTraceThreads];
  int err = 0, visits = 0, tests = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float3 o = f3(rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]), d = f3(rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]);
    float bt = kInf, bu = 0.f, bv = 0.f;
    int best = -1;
    if (brute) {
      for (int j = 0; j < s.nf; ++j) {
        const float4* tr = s.tris + 3 * (size_t)j;
        float4 a = tr[0], b = tr[1], c = tr[2];
        float t, u, v;
        if (intersect_tri(o, d, f3(a), f3(b), f3(c), t_lo, t, u, v)) {
          int id = __float_as_int(a.w);
          if (t < bt || (t == bt && id < best)) { bt = t; bu = u; bv = v; best = id; }
        }
      }
    } else {
      best = traverse(s, o, d, t_lo, bt, bu, bv, sstack + threadIdx.x, kTraceThreads, err, visits, tests);
    }
    face[i] = best;
    tuv[3 * i] = best >= 0 ? bt : 0.f;
    tuv[3 * i + 1] = bu;
    tuv[3 * i + 2] = bv;
  }
  if (err) *err_flag = 1;
}

int persistent_blocks(const void* fn, int threads, int sm_count) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
  return std::max(1, per_sm) * sm_count;
}

}  // namespace

// persistent grid of `kernel` on this context's device, cached per context (slot of grid_cache)
int cached_grid(int* cache, int slot, const void* kernel, int threads, int sm_count) {
  if (!cache[slot]) cache[slot] = persistent_blocks(kernel, threads, sm_count);
  return cache[slot];
}

cudaError_t launch_trace_primary(const FwdLaunch& a, int max_depth, int sm_count, cudaStream_t st) {
  const bool vol = a.s.env_kind == 2;
  auto kern = vol ? k_trace_primary<true> : k_trace_primary<false>;
  const int g = cached_grid(a.grids, vol ? kGridPrimaryVol : kGridPrimary, (const void*)kern, kTraceThreads, sm_count);
  kern<<<g, kTraceThreads, 0, st>>>(a, max_depth);
  return cudaGetLastError();
}

// k_shade_level<ABS, VOL>: absorption kind and volumetric env are compile-time so each
// variant carries only its own registers
template <int ABS>
void shade_dispatch(const FwdLaunch& a, int level, int max_depth, int sm_count, cudaStream_t st) {
  const bool vol = a.s.env_kind == 2;
  auto kern = ABS == 1   ? (vol ? k_shade_level_grid<true> : k_shade_level_grid<false>)
              : ABS == 2 ? (vol ? k_shade_level_hash<true> : k_shade_level_hash<false>)
              : vol      ? k_shade_level_vol
                         : k_shade_level<0, false>;
  const int g = cached_grid(a.grids, kGridShade + 2 * ABS + vol, (const void*)kern, kTraceThreads, sm_count);
  kern<<<g, kTraceThreads, 0, st>>>(a, level, max_depth);
}

cudaError_t launch_shade_level(const FwdLaunch& a, int level, int max_depth, int sm_count, cudaStream_t st) {
  if (a.s.abs_kind == 0) shade_dispatch<0>(a, level, max_depth, sm_count, st);
  else if (a.s.abs_kind == 1) shade_dispatch<1>(a, level, max_depth, sm_count, st);
  else shade_dispatch<2>(a, level, max_depth, sm_count, st);
  return cudaGetLastError();
}

cudaError_t launch_traverse_level(const FwdLaunch& a, int level, int sm_count, cudaStream_t st) {
  const int g = cached_grid(a.grids, kGridTrav, (const void*)k_traverse_level, kTraceThreads, sm_count);
  k_traverse_level<<<g, kTraceThreads, 0, st>>>(a, level);
  return cudaGetLastError();
}

cudaError_t launch_gather_level(const FwdLaunch& a, int level, int sm_count, cudaStream_t st) {
  k_gather<<<sm_count * 8, 256, 0, st>>>(a, level);
  return cudaGetLastError();
}

template <int ABS>
void backward_dispatch(const BwdLaunch& a, int level, int sm_count, cudaStream_t st) {
  const bool vol = a.s.env_kind == 2;
  auto kern = ABS == 1 ? (vol ? k_backward_level_grid<true> : k_backward_level_grid<false>)
               : ABS == 2 ? (vol ? k_backward_level_hash<true> : k_backward_level_hash<false>)
                          : (vol ? k_backward_level_vol : k_backward_level_const);
  const int g = cached_grid(a.grids, kGridBwd + 2 * ABS + vol, (const void*)kern, kBwdThreads, sm_count);
  kern<<<g, kBwdThreads, 0, st>>>(a, level, a.s.max_depth, a.cap);
}

cudaError_t launch_backward_level(const BwdLaunch& a, int level, int sm_count, cudaStream_t st) {
  if (a.s.abs_kind == 0) backward_dispatch<0>(a, level, sm_count, st);
  else if (a.s.abs_kind == 1) backward_dispatch<1>(a, level, sm_count, st);
  else backward_dispatch<2>(a, level, sm_count, st);
  return cudaGetLastError();
}

cudaError_t launch_vertex_normal_backward(dt_ctx* c, cudaStream_t st) {
  int gv = std::min((c->nv + 255) / 256, c->sm_count * 8), gf = std::min((c->nf + 255) / 256, c->sm_count * 8);
  k_vn_bwd_vertex<<<gv, 256, 0, st>>>(c->gN, c->nrm, c->nv, c->gS);
  k_vn_bwd_face<<<gf, 256, 0, st>>>(c->V, c->F, c->fnrm, c->gS, c->nf, c->fe);
  k_vn_bwd_gather<<<gv, 256, 0, st>>>(c->vstart, c->vcorner, c->fe, c->nv, c->gVn);
  return cudaGetLastError();
}

cudaError_t launch_finalize(dt_ctx* c, float* grad_V, float* grad_ior, float* grad_sigma, int accumulate,
                            cudaStream_t st) {
  int gv = std::min((c->nv + 255) / 256, c->sm_count * 8);
  if (grad_V) k_finalize<<<gv, 256, 0, st>>>(c->gV, c->gVn, c->nv, grad_V, accumulate);
  if (grad_ior) k_copy_add<<<1, 32, 0, st>>>(c->gior, grad_ior, 1, accumulate);
  if (grad_sigma) {
    int64_t n = (int64_t)c->sigma_len / 3;
    k_unpack_add<<<(int)std::min<int64_t>((n + 255) / 256, c->sm_count * 8), 256, 0, st>>>(c->gsig, grad_sigma, n,
                                                                                           accumulate);
  }
  return cudaGetLastError();
}

cudaError_t launch_loss_color(const float* rgb, const float* tgt, int64_t n, float* grad, float* loss, cudaStream_t st) {
  cudaMemsetAsync(loss, 0, sizeof(float), st);
  int g = (int)std::min<int64_t>((3 * n + 255) / 256, 148 * 16);
  k_loss_color<<<std::max(g, 1), 256, 0, st>>>(rgb, tgt, n, 1.0f / (float)std::max<int64_t>(n, 1), grad, loss);
  return cudaGetLastError();
}

cudaError_t launch_debug_closest_hit(const DevScene& s, const float* rays, int64_t n, float t_lo, int brute, int* face,
                                     float* tuv, int* err_flag, cudaStream_t st) {
  int g = (int)std::min<int64_t>((n + kTraceThreads - 1) / kTraceThreads, 148 * 32);
  k_debug_hit<<<std::max(g, 1), kTraceThreads, 0, st>>>(s, rays, n, t_lo, brute, face, tuv, err_flag);
  return cudaGetLastError();
}

cudaError_t launch_pack_sigma(const float* in, float4* out, int64_t nodes, int res, bool pairs, cudaStream_t st) {
  int g = (int)std::min<int64_t>((nodes + 255) / 256, 148 * 16);
  k_pack_sigma<<<std::max(g, 1), 256, 0, st>>>(in, out, nodes, std::max(res, 1), pairs ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_count_segments(const int* lvl, int max_depth, unsigned long long* seg, cudaStream_t st) {
  k_count_segments<<<1, 1, 0, st>>>(lvl, max_depth, seg);
  return cudaGetLastError();
}

cudaError_t launch_normals_to_f32(const D4* nrm, int nv, float* out, cudaStream_t st) {
  k_normals_to_f32<<<std::max(1, std::min((nv + 255) / 256, 148 * 8)), 256, 0, st>>>(nrm, nv, out);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const float* x, int64_t n, int* flag, cudaStream_t st) {
  int g = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_check_finite<<<std::max(g, 1), 256, 0, st>>>(x, n, flag);
  return cudaGetLastError();
}

DT_DEFINE_CHECK_READER(check_status_trace)

}  // namespace dt
