// Host-side context and kernel-launcher declarations of libdifftrans.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/difftrans.h"
#include "dt_device.cuh"

namespace dt {

// Path-record arena: one entry per traced segment, structure-of-arrays of 32-B (float64 ray
// state) and 16-B lanes so every kernel's loads/stores are coalesced vector accesses.  Levels
// (depths) are contiguous: level k occupies [off_k, off_k + cnt_k).
struct Records {
  Vec64* o;      // origin.xyz (float64), .i = ray index
  Vec64* d;      // direction.xyz (float64), .u = tree position (root 1, reflect 2p, refract 2p+1)
  float4* thr;   // throughput into the node (product of ancestors' R/T and tau), scalar R/T weight
                 //   (after the shade of a hit: the face's vertex index i2 in w)
  float4* hit;   // traversal: face, vertex indices i0 i1 i2 (int bits); after the shade:
                 //   i0, i1 (int bits), R, flags (int bits, RF_*); a miss: -1, 0, 0, RF_MISS
  float4* tau;   // interior transmittance of this segment (rgb), refract child index (int bits)
  float4* lsub;  // radiance returned by the subtree (rgb), reflect child index (int bits)
  float4* go;    // backward: dL/d(origin) of this segment, for the parent
  float4* gd;    // backward: dL/d(direction)
  float4* mq;    // volumetric env only (else null): the forward's volume moments Qc | od_M
  float4* mg;    //   and Go (env_volume), read by every backward of that forward
};
constexpr int kRecordBytes = 2 * 32 + 6 * 16;

// device int block: per-level counts and work counters
enum {
  LV_CNT = 0,            // [16] records per level
  LV_WORK_TRACE = 16,    // [16]
  LV_WORK_BWD = 32,      // [16] backward window counters (reset by every dt_trace_backward)
  LV_WORK_SHADE = 48,    // [16]
  LV_OVERFLOW = 64,
  LV_STACKERR = 65,
  LV_TRACED = 66,        // primaries traversed (passed the root-box test)
  LV_NONFINITE = 67,
  LV_WORK_PRIMARY = 68,
  LV_INTS = 80
};

// slots of dt_ctx::grid_cache
// (shade / backward: 6 slots each, by absorption kind x volumetric env)
enum { kGridPrimary = 0, kGridPrimaryVol = 1, kGridTrav = 2, kGridWide = 3, kGridShade = 4, kGridBwd = 10,
       kGridCount = 16 };

struct FwdLaunch {
  DevScene s;
  Records r;
  int* lvl;
  int64_t cap;
  float t_eps;
  // cameras
  const float* K;
  const float* c2w;
  int W, H, n_views;
  const int64_t* pids;
  int64_t n_items;      // work items for level 0
  int tiles_x, tiles_per_view;
  // tile shards (dt_cameras.tile > 0): tile side, tiles per row / per view, cyclic rule or list
  int shard_tile, stiles_x, stiles_per_view, shard_rank, shard_count;
  const int* tile_ids;
  // outputs
  float* rgb;
  float* capw;
  unsigned long long* sig_t;
  unsigned long long* sig_f;
  unsigned long long* counters;   // [0] node visits, [1] triangle tests
  int* grids;           // host: the context's persistent-grid cache (dt_ctx::grid_cache)
  int* segc;            // optional [n_rays] traced segments per ray (accumulated)
};

struct BwdLaunch {
  DevScene s;
  Records r;
  int* lvl;
  int64_t cap;
  float t_eps;
  const float* grad_rgb;
  float4* dV;       // [nv] vertex-position adjoints (atomics)
  float4* dN;       // [nv] vertex-normal adjoints (atomics)
  float4* dsig;     // [1] or [R^3] (rgb + pad)
  float* dior;      // [1]
  int* grids;       // host: the context's persistent-grid cache
};

}  // namespace dt

struct dt_ctx {
  int device = 0;
  int sm_count = 148;
  std::string err;
  // mesh snapshot
  int nv = 0, nf = 0;
  bool built = false;
  size_t cap_nv = 0, cap_nf = 0;
  float4* V = nullptr;        // [nv]
  int* F = nullptr;           // [nf*3]
  D4* nrm = nullptr;          // [nv] vertex normals (float64), |sum| in w
  D4* fnrm = nullptr;         // [nf] unit face normals (float64), |e1 x e2| in w
  // LBVH
  float4* nodes = nullptr;    // [(nf-1)*4]
  float4* tris = nullptr;     // [nf*3]
  unsigned* keys = nullptr;   // [2 * max(nf, 3nf)] radix sort ping-pong
  unsigned* vals = nullptr;
  unsigned* hist = nullptr;
  unsigned* scan_part = nullptr;   // multi-block scan chunk totals
  unsigned long long* wqueue = nullptr;   // surface-area collapse work queue (+16 ints of counters)
  int wqueue_cap = 0;
  int2* children = nullptr;   // [nf-1]
  int* parent_int = nullptr;  // [nf-1]
  int* parent_leaf = nullptr; // [nf]
  int* rflags = nullptr;      // [nf-1]
  float4* nodebox = nullptr;  // [2*(nf-1)]
  float4* leafbox = nullptr;  // [2*nf]
  int* vstart = nullptr;      // [nv+1] CSR of (vertex -> incident corners)
  unsigned* vcorner = nullptr;// [3nf] sorted corner ids (face*3 + k)
  int2* ranges = nullptr;     // [nf-1] leaf range of each binary node
  float4* wbox = nullptr;     // [2 * n_wide] wide-node boxes (checks)
  int* wdepth = nullptr;      // [n_wide] wide-node depth (checks)
  int4* went = nullptr;       // [3 (nf-1)] SAH collapse entry lists per binary node (bvh.cu)
  float* scal = nullptr;      // device scalars: [0..5] root box, [6] bbox diagonal
  int* iscal = nullptr;       // device ints: ordered-int bounds
  size_t hist_cap = 0;
  size_t scan_part_cap = 0;
  // record arena
  int64_t arena_cap = 0;
  bool arena_vol = false;       // arena carries the two volume-moment lanes (volumetric env)
  dt::Records rec{};
  int* lvl = nullptr;
  int* host_lvl = nullptr;    // pinned
  // last forward
  bool have_fwd = false;
  int64_t n_rays = 0;
  dt::DevScene fwd_scene{};
  float fwd_t_eps = 1e-4f;
  float4* sigma_snap = nullptr;  // [1] or [R^3] nodes, 2 float4 each: x-pairs (k_pack_sigma)
  size_t sigma_cap = 0, sigma_len = 0;   // sigma_len = caller floats (3 or 3 R^3)
  // gradients
  float4* gV = nullptr;       // [nv]
  float4* gN = nullptr;       // [nv]
  float4* gVn = nullptr;      // [nv]  vertex-normal chain, gathered per vertex
  float4* gS = nullptr;       // [nv]  d/d(sum of face normals)
  int* nbr_start = nullptr;   // [nv+1] vertex neighbour CSR (mesh regularisers)
  int* nbr_cnt = nullptr;     // [nv+1]
  int* nbr = nullptr;         // [<= 6 nf]
  int* nbr_owner = nullptr;   // [<= 6 nf] vertex of each neighbour entry
  int nbr_cap_v = 0;
  int64_t nbr_cap = 0;
  float4* fe = nullptr;       // [2nf] per-face d/de1, d/de2
  float4* gsig = nullptr;     // [1] or [R^3]: d/dsigma (rgb + pad)
  float* gior = nullptr;
  size_t gsig_cap = 0;
  int leaf_max = 1;           // triangles per wide-BVH leaf (r01 sweep of 1..4: 1 is fastest)
  int treelet_passes = 2;     // treelet restructuring passes per build (dt_set_bvh_quality)
  int grid_cache[dt::kGridCount] = {};    // persistent-kernel grid sizes of this device (occupancy x SMs), by kGrid*
  // profiling (dt_set_profiling / dt_get_profile)
  bool prof = false;
  double ph_ms[DT_PH_COUNT] = {};
  long long ph_launches[DT_PH_COUNT] = {};
  long long kernel_launches = 0;
  unsigned long long* counters = nullptr;       // device [8]: visits, tests (secondary), visits, tests
                                                //   (camera rays), segments
  // last forward's wavefront readback (host_lvl) and the asynchronous-forward state
  int last_D = 0, last_retries = 0;
  int64_t last_rays = 0, last_need = 0;
  bool async_pending = false;
  bool graph_fwd = false;        // the last forward was captured into a CUDA graph: host_lvl is
                                 // refreshed by each replay (read after the caller synchronises)
  cudaEvent_t fwd_done = nullptr;
  unsigned* scratch = nullptr;                  // device [16] (AdamUniform max)
  struct Pending { int ph; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
};

// Brackets one phase's launches with CUDA events on `st` when profiling is on.
struct PhaseTimer {
  dt_ctx* c;
  int ph;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  PhaseTimer(dt_ctx* c_, int ph_, cudaStream_t st_);
  void end(int n_launches);
};

// kernel launchers (bvh.cu, trace.cu)
namespace dt {
// each launcher returns the CUDA error and adds the number of kernels it launched to *nl
cudaError_t build_bvh(dt_ctx* c, const float* V, int nv, const int* F, int nf, cudaStream_t st, int* nl);
cudaError_t launch_trace_primary(const FwdLaunch& a, int max_depth, int sm_count, cudaStream_t st);
cudaError_t launch_shade_level(const FwdLaunch& a, int level, int max_depth, int sm_count, cudaStream_t st);
cudaError_t launch_traverse_level(const FwdLaunch& a, int level, int sm_count, cudaStream_t st);
cudaError_t launch_gather_level(const FwdLaunch& a, int level, int sm_count, cudaStream_t st);
cudaError_t launch_backward_level(const BwdLaunch& a, int level, int sm_count, cudaStream_t st);
cudaError_t launch_vertex_normal_backward(dt_ctx* c, cudaStream_t st);
cudaError_t launch_mesh_regularizers(dt_ctx* c, float lambda_edge, float lambda_lap, float* grad_V, float* loss,
                                     cudaStream_t st, int* nl);
cudaError_t launch_mask_loss(dt_ctx* c, const dt_cameras* cams, const float* gt, float lambda, float* grad_V,
                             float* loss, float* mask_out, cudaStream_t st, int* nl);
DevScene scene_from_ctx(const dt_ctx* c);
cudaError_t launch_finalize(dt_ctx* c, float* grad_V, float* grad_ior, float* grad_sigma, int accumulate,
                            cudaStream_t st);
cudaError_t launch_loss_color(const float* rgb, const float* tgt, int64_t n, float* grad, float* loss, cudaStream_t st);
cudaError_t launch_debug_closest_hit(const DevScene& s, const float* rays, int64_t n, float t_lo, int brute, int* face,
                                     float* tuv, int* err_flag, cudaStream_t st);
cudaError_t launch_bvh_check(dt_ctx* c, long long* out_dev, cudaStream_t st);
cudaError_t launch_normals_to_f32(const D4* nrm, int nv, float* out, cudaStream_t st);
// bounds-checked build (DT_CHECKED): first failed check line per translation unit, cleared
int check_status_bvh();
int check_status_trace();
int check_status_optim();
int check_status_meshreg();
cudaError_t launch_check_finite(const float* x, int64_t n, int* flag, cudaStream_t st);
cudaError_t launch_pack_sigma(const float* in, float4* out, int64_t nodes, int res, bool pairs, cudaStream_t st);
cudaError_t launch_count_segments(const int* lvl, int max_depth, unsigned long long* seg, cudaStream_t st);
// optim.cu
cudaError_t launch_loss_rt(const float* rgb, const float* tgt, const float* mask, int64_t n, float lc, float lt,
                           float* grad, float* loss, cudaStream_t st);
cudaError_t launch_sigma_reg(const dt_absorption* ab, const float* pts, const float* xi, int64_t n, float ls, float lv,
                             float* gsig, float* loss, cudaStream_t st);
cudaError_t launch_adam(float* p, const float* g, float* m, float* v, int64_t n, const dt_adam* c, unsigned* scratch,
                        cudaStream_t st, int* nl);
}  // namespace dt
dt_status consume_async(dt_ctx* c);
