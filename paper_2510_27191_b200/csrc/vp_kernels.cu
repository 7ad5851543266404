// vp_kernels.cu -- B200 (sm_100a) kernels of the PORPP planning step and the
// C ABI declared in include/vpb200.h.
//
// Two execution paths share the phase functions of vp_phases.cuh:
//  * vp_plan: ONE persistent cooperative kernel per planning step
//    (solver.py:79-113): tree reset, and per iteration the root draw, the
//    d_max search levels and the d_max backup levels, separated by grid
//    barriers.  Rows waiting for a node id published by the preceding
//    numbering phase spin on the hash slot instead of taking a barrier, so a
//    search level costs two grid barriers.
//  * the API kernels (vp_search / vp_backup / hooks): one launch per phase.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "vp_common.cuh"
#include "vp_models.cuh"
#include "vp_phases.cuh"

namespace cg = cooperative_groups;

namespace vp {

static thread_local cudaError_t g_last_cuda = cudaSuccess;

// ================================================================== standalone kernels (API path)

template <class PsiT, bool Exact>
__global__ void k_tree_init(vp_tree T) {
  block_tree_init<PsiT, Exact>(T);
}

__global__ void k_rehash(vp_tree T) {
  const int na = T.counters[1], nb = T.counters[0];
  const int total = na + nb;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    if (i < na) {
      const u64 key = ((u64)(u32)T.a_parent_belief[i] << 32) | (u32)T.a_action[i];
      put_final(slots(T.hash_a), T.hmask_a, key, (u32)i);
    } else {
      const int b = i - na;
      if (b == 0) continue;
      const u64 key = ((u64)(u32)T.b_parent_action[b] << 32) | T.b_parent_obs[b];
      put_final(slots(T.hash_b), T.hmask_b, key, (u32)b);
    }
  }
}

template <class Model>
__global__ void k_draw(vp_work W, const typename Model::State* particles, const double* cumw, int m, u64 key,
                       const u64* key_dev) {
  phase_draw<Model>(W, particles, cumw, m, key_dev ? *key_dev : key, this_span());
}

__device__ __forceinline__ LevelArgs level_args(const vp_search_args& S, int level, u32 stamp) {
  LevelArgs L;
  L.level = level;
  L.depth0 = S.depth0;
  L.lkey = fold(S.search_key_dev ? *S.search_key_dev : S.search_key, (u64)level);  // search.py:107
  L.stamp = stamp;
  L.inject = S.inject_actions;
  L.start = S.start_beliefs;
  return L;
}

template <class PsiT>
__device__ __forceinline__ Stage<PsiT> make_stage(unsigned char* smem, u64* bars, StageCfg cfg) {
  const int warp = threadIdx.x >> 5;
  Stage<PsiT> sg;
  sg.buf = reinterpret_cast<PsiT*>(smem) + (size_t)warp * cfg.rows * cfg.stride;
  sg.bar = &bars[warp];
  sg.phase = 0;
  sg.cfg = cfg;
  if (lane_id() == 0) {
    mbar_init(sg.bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  return sg;
}

template <class Model, class PsiT>
__global__ void __launch_bounds__(128) k_level_sample(vp_tree T, vp_model M, vp_work W, vp_search_args S, int level,
                                                      u32 stamp, StageCfg sc) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) u64 s_bar[4];
  Stage<PsiT> sg = make_stage<PsiT>(smem_raw, s_bar, sc);
  PsiT* init_cdf = reinterpret_cast<PsiT*>(smem_raw) + (size_t)4 * sc.rows * sc.stride;
  phase_sample_fast<Model, PsiT>(T, M, W, level_args(S, level, stamp), sg, init_cdf, this_span());
}

template <class Model>
__global__ void __launch_bounds__(128) k_level_sample_exact(vp_tree T, vp_model M, vp_work W, vp_search_args S,
                                                            int level, u32 stamp) {
  phase_sample_exact<Model>(T, M, W, level_args(S, level, stamp), this_span());
}

template <int WhichTable>
__global__ void __launch_bounds__(VP_SCAN_TILE) k_assign(vp_tree T, vp_work W, int level, u32 epoch) {
  phase_assign<WhichTable>(T, W, level, epoch, W.scan_ticket);
}

__global__ void __launch_bounds__(128) k_accum_probe(vp_tree T, vp_work W, int level, u32 stamp) {
  phase_accum(T, W, level, stamp, this_span());
}

template <class Model>
__global__ void __launch_bounds__(128) k_leaf(vp_tree T, vp_model M, vp_work W, vp_search_args S, int dmax,
                                              u32 stamp) {
  phase_leaf<Model>(T, M, W, level_args(S, dmax, stamp), this_span());
}

template <class PsiT>
__global__ void k_backup_leaves(vp_tree T, vp_work W, int dmax, int mat) {
  phase_backup_leaves<PsiT>(T, W, dmax, mat, this_span());
}

template <class PsiT>
__global__ void k_materialise(vp_tree T, vp_work W, int lvl) {
  phase_materialise<PsiT>(T, W, lvl, this_span());
}

template <class PsiT>
__global__ void k_backup_q(vp_tree T, vp_work W, int lvl, double gamma) {
  phase_backup_q<PsiT>(T, W, lvl, gamma, this_span());
}

template <class PsiT, bool Exact>
__global__ void k_backup_v(vp_tree T, vp_work W, int lvl, int mat) {
  phase_backup_v<PsiT, Exact>(T, W, lvl, mat, this_span());
}

__global__ void k_parent_lists(vp_tree T, vp_work W, int d, u32 stamp) {
  phase_parent_lists(T, W, d, stamp, this_span());
}

template <class PsiT>
__global__ void k_root_argmax(vp_tree T, int* out) {
  warp_root_argmax<PsiT>(T, out);
}

__global__ void k_copy_counters(vp_tree T, int* out) {
  if (threadIdx.x < 3) out[1 + threadIdx.x] = T.counters[threadIdx.x];
}

// ================================================================== persistent planning kernel

struct PlanParams {
  vp_tree T;
  vp_model M;
  vp_work W;
  int iterations, d_max_cap, m;
  double gamma;
  const void* particles;
  const double* cumw;
  const u64* keys;  // [2 * iterations]: (draw key, search key) per iteration
  int* out;         // [4]
  StageCfg sc;
  u64* timeline;    // optional: globaltimer at each phase boundary (block 0)
  int timeline_cap;
};

__device__ __forceinline__ u64 global_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One whole fixed-iteration planning step.  Barrier pattern per iteration
// with d = d_max:  draw | A(0) | B(0) C(0) | D(0) A(1) | ... | D(d-1) leaf |
// backup leaves | (Q | V |) x d, where B/D number new nodes, C/A(next)/leaf
// spin on the ids they publish, and Q/V are the backup's action and belief
// halves of each level.
template <class Model, class PsiT, bool Exact>
__global__ void __launch_bounds__(kStageWarps * 32) k_plan(PlanParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) u64 s_bar[kStageWarps];
  cg::grid_group grid = cg::this_grid();
  // grid barrier + gpu-scope fence: the fence also invalidates this SM's L1
  // (CCTL.IVALL), so plain loads after the barrier never hit lines cached
  // before another SM rewrote them (e.g. a lazily materialised PSI row that
  // shares a 128-B line with a row read earlier).
  auto barrier = [&]() {
    grid.sync();
    __threadfence();
  };
  const vp_tree& T = P.T;
  const vp_work& W = P.W;
  const Span sp = this_span();
  const int L = W.max_levels;
  Stage<PsiT> sg = make_stage<PsiT>(smem_raw, s_bar, P.sc);
  PsiT* init_cdf = reinterpret_cast<PsiT*>(smem_raw) + (size_t)kStageWarps * P.sc.rows * P.sc.stride;
  typedef typename Model::State State;

  int tl = 0;
  auto mark = [&]() {
    if (P.timeline && blockIdx.x == 0 && threadIdx.x == 0 && tl < P.timeline_cap) P.timeline[tl++] = global_ns();
  };
  mark();
  if (blockIdx.x == 0) block_tree_init<PsiT, Exact>(T);
  int d = 1;
  for (int it = 0; it < P.iterations; ++it) {
    const u32 stamp_base = (u32)it * (u32)(L + 3);
    const u64 skey = P.keys[2 * it + 1];
    if (sp.gtid <= d) W.fcount[sp.gtid] = 0;
    if (sp.gtid < d) W.pcount[sp.gtid] = 0;
    phase_draw<Model>(W, reinterpret_cast<const State*>(P.particles), P.cumw, P.m, P.keys[2 * it], sp);
    barrier();
    mark();
    for (int l = 0; l < d; ++l) {
      LevelArgs la;
      la.level = l;
      la.depth0 = 0;
      la.lkey = fold(skey, (u64)l);
      la.stamp = stamp_base + (u32)l + 1u;
      la.inject = nullptr;
      la.start = nullptr;
      const u32 epoch = 1u + 2u * ((u32)it * (u32)(L + 1) + (u32)l);
      if constexpr (Exact) phase_sample_exact<Model>(T, P.M, W, la, sp);
      else phase_sample_fast<Model, PsiT>(T, P.M, W, la, sg, init_cdf, sp);
      barrier();
      mark();
      phase_assign<0>(T, W, l, epoch, nullptr);
      phase_accum(T, W, l, la.stamp, sp);
      barrier();
      mark();
      phase_assign<1>(T, W, l, epoch + 1u, nullptr);
    }
    {
      LevelArgs la;
      la.level = d;
      la.depth0 = 0;
      la.lkey = 0;
      la.stamp = stamp_base + (u32)d + 1u;
      la.inject = nullptr;
      la.start = nullptr;
      phase_leaf<Model>(T, P.M, W, la, sp);
    }
    barrier();
    mark();
    phase_backup_leaves<PsiT>(T, W, d, d - 1, sp);
    barrier();
    mark();
    for (int lv = d - 1; lv >= 0; --lv) {
      phase_backup_q<PsiT>(T, W, lv, P.gamma, sp);
      barrier();
      mark();
      phase_backup_v<PsiT, Exact>(T, W, lv, lv - 1, sp);
      barrier();
      mark();
    }
    d = d + 1 < P.d_max_cap ? d + 1 : P.d_max_cap;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    warp_root_argmax<PsiT>(T, P.out);
    if (threadIdx.x < 3) P.out[1 + threadIdx.x] = T.counters[threadIdx.x];
  }
}

// ================================================================== host side

static inline int blocks_for(long long n, int bs) { return (int)((n + bs - 1) / bs); }

static int32_t check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_last_cuda = e;
    return VP_ERR_CUDA;
  }
  return VP_OK;
}

// ---- per-launch accounting: launch counter + optional CUDA-event timing by kernel kind
enum KernelKind {
  KK_DRAW = 0, KK_LEVEL_SAMPLE, KK_ASSIGN_ACTIONS, KK_ACCUM_PROBE, KK_ASSIGN_BELIEFS, KK_LEAF,
  KK_BACKUP_LEAVES, KK_BACKUP_Q, KK_BACKUP_V, KK_PARENT_LISTS, KK_ARGMAX, KK_TREE_INIT, KK_REHASH, KK_PLAN, KK_COUNT
};
struct ProfRec {
  int kind;
  cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_prof_pool;
static size_t g_prof_used = 0;
static bool g_prof_on = false;
static long long g_launches = 0;

static cudaEvent_t prof_event() {
  if (g_prof_used == g_prof_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_prof_pool.push_back(e);
  }
  return g_prof_pool[g_prof_used++];
}

struct Launch {
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Launch(int k, cudaStream_t s) : kind(k), st(s) {
    ++g_launches;
    if (g_prof_on) {
      a = prof_event();
      cudaEventRecord(a, st);
    }
  }
  ~Launch() {
    if (g_prof_on) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, st);
      g_prof_recs.push_back({kind, a, b});
    }
  }
};

template <class F>
static int32_t dispatch_model(int kind, F&& f) {
  switch (kind) {
    case VP_MODEL_MARS: return f(MarsModel());
    case VP_MODEL_TABULAR: return f(TabularModel());
    case VP_MODEL_SYNTHETIC: return f(SyntheticModel());
    case VP_MODEL_LIGHTDARK: return f(LightDarkModel());
    default: return VP_ERR_MODEL;
  }
}

template <class F>
static int32_t dispatch_psi(int dtype, int exact, F&& f) {
  if (dtype == VP_PSI_F32) {
    if (exact) return VP_ERR_INVALID;  // numpy-order parity mode is fp64 only
    return f((float)0, std::false_type());
  }
  if (dtype == VP_PSI_F64) {
    if (exact) return f((double)0, std::true_type());
    return f((double)0, std::false_type());
  }
  return VP_ERR_INVALID;
}

template <class Model>
static bool state_size_ok(const vp_model& M) {
  return M.state_bytes == (int)sizeof(typename Model::State);
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Staged-row geometry: rows padded to an odd number of 16-B chunks so the
// LDS.128 scans of 8 lanes in different rows hit different bank groups.
template <class PsiT>
static StageCfg stage_cfg(int A, int warps, int budget_bytes) {
  int chunks = (int)(((size_t)A * sizeof(PsiT) + 15) / 16);
  if ((chunks & 1) == 0) ++chunks;
  StageCfg c;
  c.stride = chunks * 16 / (int)sizeof(PsiT);
  c.rows = std::max(1, std::min(32, budget_bytes / warps / (chunks * 16)));
  return c;
}
// staged rows of every warp + the block's copy of the initial-row CDF
template <class PsiT>
static size_t stage_bytes(const StageCfg& c, int warps, int A) {
  return ((size_t)warps * c.rows * c.stride + (size_t)A) * sizeof(PsiT);
}

template <class Model, class PsiT, bool Exact>
static int32_t set_sample_attr(size_t smem) {
  if constexpr (!Exact) {
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
      if (cudaFuncSetAttribute(k_level_sample<Model, PsiT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem) != cudaSuccess)
        return VP_ERR_CUDA;
      configured = smem;
    }
  }
  return VP_OK;
}

template <class Model, class PsiT, bool Exact>
static int32_t run_search(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_search_args& S,
                          cudaStream_t st) {
  const int n = W.n;
  const int grid = blocks_for(n, 128);
  const int tiles = blocks_for(n, VP_SCAN_TILE);
  if (cudaMemsetAsync(W.fcount, 0, sizeof(int32_t) * (W.max_levels + 1), st) != cudaSuccess) return VP_ERR_CUDA;
  if (cudaMemsetAsync(W.pcount, 0, sizeof(int32_t) * W.max_levels, st) != cudaSuccess) return VP_ERR_CUDA;
  if (cudaMemsetAsync(W.scan_status, 0, sizeof(uint64_t) * tiles, st) != cudaSuccess) return VP_ERR_CUDA;
  if (cudaMemsetAsync(W.scan_ticket, 0, sizeof(uint32_t), st) != cudaSuccess) return VP_ERR_CUDA;
  StageCfg sc{0, 0};
  size_t smem = 0;
  if constexpr (!Exact) {
    sc = stage_cfg<PsiT>(T.action_count, 4, env_int("VP_STAGE_KB", 200) * 1024);
    smem = stage_bytes<PsiT>(sc, 4, T.action_count);
    if (int32_t rc = set_sample_attr<Model, PsiT, Exact>(smem)) return rc;
  }
  for (int l = S.depth0; l < S.d_max; ++l) {
    const u32 stamp = S.stamp_base + (u32)l + 1u;
    {
      Launch L_(KK_LEVEL_SAMPLE, st);
      if constexpr (Exact) k_level_sample_exact<Model><<<grid, 128, 0, st>>>(T, M, W, S, l, stamp);
      else k_level_sample<Model, PsiT><<<grid, 128, smem, st>>>(T, M, W, S, l, stamp, sc);
    }
    { Launch L_(KK_ASSIGN_ACTIONS, st); k_assign<0><<<tiles, VP_SCAN_TILE, 0, st>>>(T, W, l, (u32)(2 * l + 1)); }
    { Launch L_(KK_ACCUM_PROBE, st); k_accum_probe<<<grid, 128, 0, st>>>(T, W, l, stamp); }
    { Launch L_(KK_ASSIGN_BELIEFS, st); k_assign<1><<<tiles, VP_SCAN_TILE, 0, st>>>(T, W, l, (u32)(2 * l + 2)); }
  }
  { Launch L_(KK_LEAF, st); k_leaf<Model><<<grid, 128, 0, st>>>(T, M, W, S, S.d_max, S.stamp_base + (u32)S.d_max + 1u); }
  return check_launch();
}

template <class PsiT, bool Exact>
static int32_t run_backup(const vp_tree& T, const vp_work& W, int depth0, int dmax, double gamma, u32 stamp_base,
                          cudaStream_t st) {
  const int n = W.n;
  const int grid = blocks_for(n, 256);
  const int wgrid = std::min(blocks_for((long long)n * 32, 256), 148 * 32);
  const int vgrid = Exact ? std::max(grid, wgrid) : wgrid;
  if (dmax < 1) return VP_OK;
  // lists of level L exist (recorded by search) for depth0 <= L <= dmax
  auto recorded = [&](int L) { return L >= depth0 && L >= 0 ? L : -1; };
  { Launch L_(KK_BACKUP_LEAVES, st); k_backup_leaves<PsiT><<<wgrid, 256, 0, st>>>(T, W, dmax, recorded(dmax - 1)); }
  for (int d = dmax; d >= 1; --d) {
    if (d <= depth0) {
      if (cudaMemsetAsync(W.pcount + (d - 1), 0, sizeof(int32_t), st) != cudaSuccess) return VP_ERR_CUDA;
      if (cudaMemsetAsync(W.fcount + (d - 1), 0, sizeof(int32_t), st) != cudaSuccess) return VP_ERR_CUDA;
      { Launch L_(KK_PARENT_LISTS, st); k_parent_lists<<<grid, 256, 0, st>>>(T, W, d, stamp_base + 0x40000000u + (u32)d); }
      { Launch L_(KK_PARENT_LISTS, st); k_materialise<PsiT><<<wgrid, 256, 0, st>>>(T, W, d - 1); }
    }
    { Launch L_(KK_BACKUP_Q, st); k_backup_q<PsiT><<<grid, 256, 0, st>>>(T, W, d - 1, gamma); }
    { Launch L_(KK_BACKUP_V, st); k_backup_v<PsiT, Exact><<<vgrid, 256, 0, st>>>(T, W, d - 1, d >= 2 ? recorded(d - 2) : -1); }
  }
  return check_launch();
}

// ---- whole planning step

template <class Model, class PsiT, bool Exact>
static int32_t enqueue_inputs(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_plan_args& P,
                              cudaStream_t st) {
  typedef typename Model::State State;
  if (P.keys_host &&
      cudaMemcpyAsync(P.keys_dev, P.keys_host, 16 * (size_t)P.iterations, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return VP_ERR_CUDA;
  if (P.particles_host && cudaMemcpyAsync(P.particles_dev, P.particles_host, (size_t)P.m * sizeof(State),
                                          cudaMemcpyHostToDevice, st) != cudaSuccess)
    return VP_ERR_CUDA;
  if (P.cumw_host &&
      cudaMemcpyAsync(P.cumw_dev, P.cumw_host, 8 * (size_t)P.m, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return VP_ERR_CUDA;
  if (cudaMemsetAsync(T.hash_a, 0xff, (T.hmask_a + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  if (cudaMemsetAsync(T.hash_b, 0xff, (T.hmask_b + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  return VP_OK;
}

// Multi-kernel version of a planning step (one launch per phase).
template <class Model, class PsiT, bool Exact>
static int32_t enqueue_plan_kernels(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_plan_args& P,
                                    cudaStream_t st) {
  typedef typename Model::State State;
  if (int32_t rc = enqueue_inputs<Model, PsiT, Exact>(T, M, W, P, st)) return rc;
  { Launch L_(KK_TREE_INIT, st); k_tree_init<PsiT, Exact><<<1, 256, 0, st>>>(T); }
  const u64* keys = reinterpret_cast<const u64*>(P.keys_dev);
  int d = 1;
  for (int it = 0; it < P.iterations; ++it) {
    // the API kernels read the keys from device memory via search_key_dev
    {
      Launch L_(KK_DRAW, st);
      k_draw<Model><<<blocks_for(W.n, 256), 256, 0, st>>>(W, reinterpret_cast<const State*>(P.particles_dev),
                                                         P.cumw_dev, P.m, 0ull, keys + 2 * it);
    }
    vp_search_args S;
    memset(&S, 0, sizeof(S));
    S.search_key_dev = P.keys_dev + 2 * it + 1;
    S.d_max = d;
    S.stamp_base = (u32)it * (u32)(W.max_levels + 3);
    S.iteration = it;
    int32_t rc = run_search<Model, PsiT, Exact>(T, M, W, S, st);
    if (rc) return rc;
    rc = run_backup<PsiT, Exact>(T, W, 0, d, P.gamma, S.stamp_base, st);
    if (rc) return rc;
    d = std::min(d + 1, P.d_max_cap);
  }
  { Launch L_(KK_ARGMAX, st); k_root_argmax<PsiT><<<1, 32, 0, st>>>(T, P.out_dev); }
  { Launch L_(KK_ARGMAX, st); k_copy_counters<<<1, 32, 0, st>>>(T, P.out_dev); }
  if (P.out_host &&
      cudaMemcpyAsync(P.out_host, P.out_dev, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return VP_ERR_CUDA;
  return check_launch();
}

static int g_num_sms = 0;

// Persistent version: inputs, tree reset, ONE cooperative kernel, result.
template <class Model, class PsiT, bool Exact>
static int32_t enqueue_plan_persistent(const vp_tree& T, const vp_model& M, const vp_work& W,
                                       const vp_plan_args& P, cudaStream_t st) {
  if (int32_t rc = enqueue_inputs<Model, PsiT, Exact>(T, M, W, P, st)) return rc;
  const int tiles = blocks_for(W.n, VP_SCAN_TILE);
  if (cudaMemsetAsync(W.scan_status, 0, sizeof(uint64_t) * tiles, st) != cudaSuccess) return VP_ERR_CUDA;
  PlanParams pp;
  pp.T = T;
  pp.M = M;
  pp.W = W;
  pp.iterations = P.iterations;
  pp.d_max_cap = P.d_max_cap;
  pp.m = P.m;
  pp.gamma = P.gamma;
  pp.particles = P.particles_dev;
  pp.cumw = P.cumw_dev;
  pp.keys = reinterpret_cast<const u64*>(P.keys_dev);
  pp.out = P.out_dev;
  pp.timeline = reinterpret_cast<u64*>(P.timeline_dev);
  pp.timeline_cap = P.timeline_cap;
  pp.sc = Exact ? StageCfg{1, 4} : stage_cfg<PsiT>(T.action_count, kStageWarps, env_int("VP_PLAN_STAGE_KB", 96) * 1024);
  const size_t smem = Exact ? 16 : stage_bytes<PsiT>(pp.sc, kStageWarps, T.action_count);
  auto kern = k_plan<Model, PsiT, Exact>;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return check_launch();
    configured = smem;
  }
  if (!g_num_sms) cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, 0);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStageWarps * 32, smem) != cudaSuccess ||
      per_sm < 1)
    return check_launch();
  per_sm = std::min(per_sm, env_int("VP_PLAN_BLOCKS_PER_SM", 4));
  const int grid = std::max(1, g_num_sms * per_sm);
  void* args[] = {&pp};
  {
    Launch L_(KK_PLAN, st);
    if (cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kStageWarps * 32), args, smem, st) !=
        cudaSuccess)
      return check_launch();
  }
  if (P.out_host &&
      cudaMemcpyAsync(P.out_host, P.out_dev, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return VP_ERR_CUDA;
  return check_launch();
}

struct GraphEntry {
  std::vector<unsigned char> key;
  cudaGraphExec_t exec;
  long long launches;
  unsigned long long used;
};
static std::vector<GraphEntry> g_graphs;
static unsigned long long g_graph_clock = 0;
static cudaStream_t g_capture_stream = nullptr;

template <class T>
static void append_pod(std::vector<unsigned char>& v, const T& x) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(&x);
  v.insert(v.end(), p, p + sizeof(T));
}

// mode 0: multi-kernel direct; 1: multi-kernel captured into a CUDA graph
// (replayed while pointers / sizes / model are unchanged); 2: persistent.
template <class Model, class PsiT, bool Exact>
static int32_t run_plan(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_plan_args& P,
                        cudaStream_t st) {
  if (P.mode == 2) return enqueue_plan_persistent<Model, PsiT, Exact>(T, M, W, P, st);
  if constexpr (!Exact) {
    const StageCfg sc = stage_cfg<PsiT>(T.action_count, 4, env_int("VP_STAGE_KB", 200) * 1024);
    if (int32_t rc = set_sample_attr<Model, PsiT, Exact>(stage_bytes<PsiT>(sc, 4, T.action_count))) return rc;
  }
  if (P.mode == 0 || g_prof_on) return enqueue_plan_kernels<Model, PsiT, Exact>(T, M, W, P, st);
  std::vector<unsigned char> key;
  append_pod(key, T);
  append_pod(key, M);
  append_pod(key, W);
  append_pod(key, P);
  const int budget = env_int("VP_STAGE_KB", 200);
  append_pod(key, budget);
  GraphEntry* hit = nullptr;
  for (auto& e : g_graphs)
    if (e.key == key) hit = &e;
  if (!hit) {
    if (!g_capture_stream && cudaStreamCreateWithFlags(&g_capture_stream, cudaStreamNonBlocking) != cudaSuccess)
      return VP_ERR_CUDA;
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, st);
    cudaStreamWaitEvent(g_capture_stream, ev, 0);
    cudaEventDestroy(ev);
    cudaStreamSynchronize(g_capture_stream);
    const long long l0 = g_launches;
    if (cudaStreamBeginCapture(g_capture_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return VP_ERR_CUDA;
    int32_t rc = enqueue_plan_kernels<Model, PsiT, Exact>(T, M, W, P, g_capture_stream);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(g_capture_stream, &graph);
    const long long launches = g_launches - l0;
    g_launches = l0;
    if (rc || ce != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      g_last_cuda = ce;
      return rc ? rc : VP_ERR_CUDA;
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      g_last_cuda = ie;
      return VP_ERR_CUDA;
    }
    if (g_graphs.size() >= 16) {
      size_t lru = 0;
      for (size_t i = 1; i < g_graphs.size(); ++i)
        if (g_graphs[i].used < g_graphs[lru].used) lru = i;
      cudaGraphExecDestroy(g_graphs[lru].exec);
      g_graphs.erase(g_graphs.begin() + lru);
    }
    g_graphs.push_back(GraphEntry{key, exec, launches, 0});
    hit = &g_graphs.back();
  }
  hit->used = ++g_graph_clock;
  if (cudaGraphLaunch(hit->exec, st) != cudaSuccess) return check_launch();
  g_launches += hit->launches;
  return check_launch();
}

// ---- test-hook kernels

__global__ void k_rng_uniform(u64 key, const int64_t* rows, int64_t n, int k, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 r = (u64)rows[i];
  if (k <= 0) out[i] = uniform1(key, r);
  else
    for (int j = 1; j <= k; ++j) out[i * k + (j - 1)] = uniform_j(key, r, (u64)j);
}
__global__ void k_rng_normal(u64 key, const int64_t* rows, int64_t n, int k, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 r = (u64)rows[i];
  if (k <= 0) out[i] = normal_j(key, r, 0);
  else
    for (int j = 1; j <= k; ++j) out[i * k + (j - 1)] = normal_j(key, r, (u64)j);
}
template <class Model>
__global__ void k_model_step(vp_model M, typename Model::State* st, const int32_t* act, u64 key,
                             const int64_t* rows, int n, u32* obs, double* rew) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  typename Model::State s = st[i];
  u32 o;
  double r;
  Model::step(M, s, act[i], key, (u64)rows[i], o, r);
  st[i] = s;
  obs[i] = o;
  rew[i] = r;
}
template <class Model>
__global__ void k_model_heur(vp_model M, const typename Model::State* st, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = Model::heuristic(M, st[i]);
}
template <class PsiT, bool Exact>
__global__ void k_lse_rows(const PsiT* rows, int count, int width, double eta, double* out) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= count) return;
  if constexpr (Exact) {
    if (lane_id() == 0) out[gw] = lse_exact(reinterpret_cast<const double*>(rows) + (size_t)gw * width, width, eta);
  } else {
    const double v = row_lse_fast<PsiT>(rows + (size_t)gw * width, width, eta);
    if (lane_id() == 0) out[gw] = v;
  }
}
template <class PsiT, bool Exact>
__global__ void k_sample_rows(const PsiT* rows, int width, double eta, const double* lse, const int32_t* group,
                              const double* u, int n, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int g = group[i];
  if constexpr (Exact) {
    out[i] = sample_exact(reinterpret_cast<const double*>(rows) + (size_t)g * width, width, eta, u[i]);
  } else {
    const PsiT e2 = (PsiT)(eta * kLog2eD), sh2 = (PsiT)(eta * lse[g] * kLog2eD);
    out[i] = scan_cdf_scalar<PsiT>(rows + (size_t)g * width, width, e2, sh2, (PsiT)u[i]);
  }
}

}  // namespace vp

// ================================================================== C ABI

using namespace vp;

extern "C" {

int32_t vp_abi_version(void) { return VPB200_ABI_VERSION; }

const char* vp_status_string(int32_t s) {
  switch (s) {
    case VP_OK: return "ok";
    case VP_ERR_INVALID: return "invalid argument";
    case VP_ERR_CAPACITY: return "capacity exceeded";
    case VP_ERR_CUDA: return cudaGetErrorString(g_last_cuda);
    case VP_ERR_MODEL: return "unsupported model kind";
    default: return "unknown status";
  }
}

int32_t vp_last_cuda_error(void) { return (int32_t)g_last_cuda; }

int32_t vp_profile_enable(int32_t on) {
  g_prof_on = on != 0;
  if (g_prof_on) {
    g_prof_recs.clear();
    g_prof_used = 0;
  }
  return VP_OK;
}

int32_t vp_profile_read(double* ms_by_kind, int64_t* launches_by_kind, int32_t nkinds) {
  if (!ms_by_kind || !launches_by_kind) return KK_COUNT;
  for (int i = 0; i < nkinds; ++i) {
    ms_by_kind[i] = 0.0;
    launches_by_kind[i] = 0;
  }
  for (const ProfRec& r : g_prof_recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return VP_ERR_CUDA;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (r.kind < nkinds) {
      ms_by_kind[r.kind] += ms;
      launches_by_kind[r.kind] += 1;
    }
  }
  return KK_COUNT;
}

int64_t vp_launch_count(void) { return g_launches; }

int32_t vp_abi_layout(int32_t* out, int32_t n) {
  // sizes and a few field offsets so the host binding can verify its mirror
  const int32_t v[] = {(int32_t)sizeof(vp_model),
                       (int32_t)sizeof(vp_tree),
                       (int32_t)sizeof(vp_work),
                       (int32_t)sizeof(vp_search_args),
                       (int32_t)offsetof(vp_model, tab_states),
                       (int32_t)offsetof(vp_model, ld_bins),
                       (int32_t)offsetof(vp_tree, eta),
                       (int32_t)offsetof(vp_work, trace_belief),
                       (int32_t)offsetof(vp_search_args, start_beliefs),
                       (int32_t)sizeof(Slot),
                       (int32_t)sizeof(vp_plan_args),
                       (int32_t)offsetof(vp_plan_args, out_dev),
                       (int32_t)offsetof(vp_tree, init_cdf)};
  const int32_t m = (int32_t)(sizeof(v) / sizeof(v[0]));
  if (!out) return m;
  for (int32_t i = 0; i < n && i < m; ++i) out[i] = v[i];
  return m;
}

int32_t vp_tree_init(const vp_tree* t, void* stream) {
  if (!t || t->action_count < 1) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(t->hash_a, 0xff, (t->hmask_a + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  if (cudaMemsetAsync(t->hash_b, 0xff, (t->hmask_b + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  const vp_tree T = *t;
  return dispatch_psi(T.psi_dtype, T.exact, [&](auto z, auto ex) -> int32_t {
    typedef decltype(z) PsiT;
    Launch L_(KK_TREE_INIT, st);
    k_tree_init<PsiT, decltype(ex)::value><<<1, 256, 0, st>>>(T);
    return check_launch();
  });
}

int32_t vp_tree_rehash(const vp_tree* t, void* stream) {
  if (!t) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(t->hash_a, 0xff, (t->hmask_a + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  if (cudaMemsetAsync(t->hash_b, 0xff, (t->hmask_b + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  { Launch L_(KK_REHASH, st); k_rehash<<<148 * 8, 256, 0, st>>>(*t); }
  return check_launch();
}

int32_t vp_tree_counts(const vp_tree* t, int32_t* host_out, void* stream) {
  if (!t || !host_out) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(host_out, t->counters, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return VP_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return VP_ERR_CUDA;
  return VP_OK;
}

int32_t vp_draw_root_states(const vp_model* m, const vp_work* w, const void* particles, const double* cumw,
                            int32_t count, uint64_t key, void* stream) {
  if (!m || !w || !particles || !cumw || count < 1 || w->n < 1) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_work W = *w;
  return dispatch_model(m->kind, [&](auto mdl) -> int32_t {
    typedef decltype(mdl) Model;
    if (!state_size_ok<Model>(*m)) return VP_ERR_INVALID;
    Launch L_(KK_DRAW, st);
    k_draw<Model><<<blocks_for(W.n, 256), 256, 0, st>>>(
        W, reinterpret_cast<const typename Model::State*>(particles), cumw, count, key, nullptr);
    return check_launch();
  });
}

int32_t vp_search(const vp_tree* t, const vp_model* m, const vp_work* w, const vp_search_args* a, void* stream) {
  if (!t || !m || !w || !a) return VP_ERR_INVALID;
  if (a->depth0 < 0 || a->d_max < a->depth0 || a->d_max > w->max_levels) return VP_ERR_INVALID;
  if (m->action_count != t->action_count) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_tree T = *t;
  const vp_model M = *m;
  const vp_work W = *w;
  const vp_search_args S = *a;
  return dispatch_model(M.kind, [&](auto mdl) -> int32_t {
    typedef decltype(mdl) Model;
    if (!state_size_ok<Model>(M)) return VP_ERR_INVALID;
    return dispatch_psi(T.psi_dtype, T.exact, [&](auto z, auto ex) -> int32_t {
      return run_search<Model, decltype(z), decltype(ex)::value>(T, M, W, S, st);
    });
  });
}

int32_t vp_plan(const vp_tree* t, const vp_model* m, const vp_work* w, const vp_plan_args* p, void* stream) {
  if (!t || !m || !w || !p) return VP_ERR_INVALID;
  if (p->iterations < 1 || p->d_max_cap < 1 || p->m < 1 || !p->keys_dev || !p->particles_dev || !p->cumw_dev ||
      !p->out_dev)
    return VP_ERR_INVALID;
  if (std::min(p->iterations, p->d_max_cap) > w->max_levels) return VP_ERR_INVALID;
  if (m->action_count != t->action_count) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_tree T = *t;
  const vp_model M = *m;
  const vp_work W = *w;
  const vp_plan_args P = *p;
  return dispatch_model(M.kind, [&](auto mdl) -> int32_t {
    typedef decltype(mdl) Model;
    if (!state_size_ok<Model>(M)) return VP_ERR_INVALID;
    return dispatch_psi(T.psi_dtype, T.exact, [&](auto z, auto ex) -> int32_t {
      return run_plan<Model, decltype(z), decltype(ex)::value>(T, M, W, P, st);
    });
  });
}

int32_t vp_backup(const vp_tree* t, const vp_work* w, int32_t depth0, int32_t d_max, double gamma,
                  uint32_t stamp_base, void* stream) {
  if (!t || !w || depth0 < 0 || d_max < depth0 || d_max > w->max_levels) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_tree T = *t;
  const vp_work W = *w;
  return dispatch_psi(T.psi_dtype, T.exact, [&](auto z, auto ex) -> int32_t {
    return run_backup<decltype(z), decltype(ex)::value>(T, W, depth0, d_max, gamma, stamp_base, st);
  });
}

int32_t vp_root_argmax(const vp_tree* t, int32_t* out_dev, void* stream) {
  if (!t || !out_dev) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_tree T = *t;
  return dispatch_psi(T.psi_dtype, T.exact, [&](auto z, auto) -> int32_t {
    Launch L_(KK_ARGMAX, st);
    k_root_argmax<decltype(z)><<<1, 32, 0, st>>>(T, out_dev);
    return check_launch();
  });
}

int32_t vp_rng_uniform(uint64_t key, const int64_t* rows, int64_t n, int32_t k, double* out, void* stream) {
  if (n < 0 || (n && (!rows || !out))) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  k_rng_uniform<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(key, rows, n, k, out);
  return check_launch();
}

int32_t vp_rng_normal(uint64_t key, const int64_t* rows, int64_t n, int32_t k, double* out, void* stream) {
  if (n < 0 || (n && (!rows || !out))) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  k_rng_normal<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(key, rows, n, k, out);
  return check_launch();
}

int32_t vp_model_step(const vp_model* m, void* states, const int32_t* actions, uint64_t key, const int64_t* rows,
                      int32_t n, uint32_t* obs_out, double* reward_out, void* stream) {
  if (!m || n < 0) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_model M = *m;
  return dispatch_model(M.kind, [&](auto mdl) -> int32_t {
    typedef decltype(mdl) Model;
    if (!state_size_ok<Model>(M)) return VP_ERR_INVALID;
    k_model_step<Model><<<blocks_for(n, 256), 256, 0, st>>>(
        M, reinterpret_cast<typename Model::State*>(states), actions, key, rows, n, obs_out, reward_out);
    return check_launch();
  });
}

int32_t vp_model_heuristic(const vp_model* m, const void* states, int32_t n, double* out, void* stream) {
  if (!m || n < 0) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_model M = *m;
  return dispatch_model(M.kind, [&](auto mdl) -> int32_t {
    typedef decltype(mdl) Model;
    if (!state_size_ok<Model>(M)) return VP_ERR_INVALID;
    k_model_heur<Model><<<blocks_for(n, 256), 256, 0, st>>>(
        M, reinterpret_cast<const typename Model::State*>(states), n, out);
    return check_launch();
  });
}

int32_t vp_lse_rows(const void* rows, int32_t dtype, int32_t exact, int32_t count, int32_t width, double eta,
                    double* out, void* stream) {
  if (count < 0 || width < 1 || eta <= 0) return VP_ERR_INVALID;
  if (!count) return VP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  return dispatch_psi(dtype, exact, [&](auto z, auto ex) -> int32_t {
    typedef decltype(z) PsiT;
    k_lse_rows<PsiT, decltype(ex)::value><<<blocks_for((long long)count * 32, 256), 256, 0, st>>>(
        reinterpret_cast<const PsiT*>(rows), count, width, eta, out);
    return check_launch();
  });
}

int32_t vp_sample_rows(const void* rows, int32_t dtype, int32_t exact, int32_t count, int32_t width, double eta,
                       const double* lse, const int32_t* group, const double* u, int32_t n, int32_t* out,
                       void* stream) {
  if (count < 1 || width < 1 || eta <= 0 || n < 0) return VP_ERR_INVALID;
  if (!exact && !lse) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  return dispatch_psi(dtype, exact, [&](auto z, auto ex) -> int32_t {
    typedef decltype(z) PsiT;
    k_sample_rows<PsiT, decltype(ex)::value><<<blocks_for(n, 256), 256, 0, st>>>(
        reinterpret_cast<const PsiT*>(rows), width, eta, lse, group, u, n, out);
    return check_launch();
  });
}

}  // extern "C"
