// vp_kernels.cu -- B200 (sm_100a) kernels of the PORPP planning step and the
// C ABI declared in include/vpb200.h.
//
// A planning pass (root draw + search + backup, solver.py:96-111) is two
// kernel launches with no grid barrier (vp_phases.cuh); a fixed-iteration
// planning step (vp_plan) is tree reset + 2 x iterations launches + the root
// argmax, captured once into a CUDA graph and replayed.
#include <algorithm>
#include <cfloat>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <atomic>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "vp_common.cuh"
#include "vp_models.cuh"
#include "vp_phases.cuh"

namespace vp {

static thread_local cudaError_t g_last_cuda = cudaSuccess;

// ================================================================== kernels

template <class PsiT, bool Exact>
__global__ void k_tree_init(vp_tree T) {
  block_tree_init<PsiT, Exact>(T);
}

// Tree reset, part 1: every row the previous tree used gets zero accumulators
// and an unset creation key, so node creation needs no initialising stores
// that other rows would have to wait for (rows beyond the previous counts are
// in that state since allocation).  Part 2 (k_tree_init) rewrites the root.
__global__ void k_clear(vp_tree T) {
  const int nb = min(T.counters[0], T.cap_beliefs), na = min(T.counters[VP_COUNTER_ACTIONS], T.cap_actions);
  const int nd = T.exact ? 0 : min(T.counters[VP_COUNTER_DENSE], T.cap_dense);
  const int total = max(max(nb, na), nd);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    if (i < nb) {
      T.b_value[i] = 0.0;
      T.b_rows[i] = 0;
      reinterpret_cast<Acc*>(T.b_acc)[i] = Acc{0.0, 0u, 0u};
      T.b_ckey[i] = ~0ull;
      T.b_nact[i] = 0;
      const int words = T.psi_dtype == VP_PSI_F32 ? 2 : 3;  // sizeof(Rec<PsiT>) / 16
      uint4* rec = reinterpret_cast<uint4*>(T.b_rec) + (size_t)i * words;
      for (int w = 0; w < words; ++w) rec[w] = make_uint4(0u, 0u, 0u, 0u);
    }
    if (i < nd) reinterpret_cast<uint4*>(T.dense_meta)[i] = make_uint4(0u, 0u, 0u, 0u);  // no CDF requests
    if (i < na) {
      T.a_reward[i] = 0.0;
      T.a_visits[i] = 0;
      T.a_rows[i] = 0;
      reinterpret_cast<Acc*>(T.a_acc)[i] = Acc{0.0, 0u, 0u};
      T.a_ckey[i] = ~0ull;
    }
  }
}

// eta changed on a live tree (the search / backup hooks take eta per call, search.py:86,
// backup.py:75): the initial row's LSE and CDF (one warp) and then every live row's cached
// LSE -- the initial LSE for lazily initial rows, the row's own LSE otherwise.
template <class PsiT, bool Exact>
__global__ void k_eta_init_row(vp_tree T) {
  if (threadIdx.x >= 32) return;
  const int A = T.action_count;
  PsiT* cdf = reinterpret_cast<PsiT*>(T.init_cdf);
  double v;
  if constexpr (Exact) {
    v = 0.0;
    if (threadIdx.x == 0) v = lse_exact(T.init_prefs, A, T.eta);
    v = __shfl_sync(FULL, v, 0);
  } else {
    for (int a = threadIdx.x; a < A; a += 32) cdf[a] = (PsiT)T.init_prefs[a];
    __syncwarp();
    v = row_lse_f64<PsiT>(cdf, A, T.eta);
  }
  for (int a = threadIdx.x; a < A; a += 32) cdf[a] = (PsiT)T.init_prefs[a];
  __syncwarp();
  const PsiT total = row_cdf_inplace(cdf, A, (PsiT)(T.eta * kLog2eD), (PsiT)(T.eta * v * kLog2eD));
  for (int a = threadIdx.x; a < A; a += 32) cdf[a] = cdf[a] / total;
  if (threadIdx.x == 0) T.init_lse[0] = v;
}

template <class PsiT, bool Exact>
__global__ void k_eta_rows(vp_tree T) {
  const int nb = min(T.counters[0], T.cap_beliefs);
  const int warps = gridDim.x * (blockDim.x >> 5);
  const PsiT* psi = reinterpret_cast<const PsiT*>(T.psi);
  for (int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
    double v;
    if constexpr (!Exact) {  // dense row, overlay row or the initial row
      const Rec<PsiT> r = load_rec<PsiT>(T, b);
      if (r.dense_pass) {
        v = row_lse_f64<PsiT>(psi + (size_t)r.dense_row * T.psi_stride, T.action_count, T.eta);
      } else if (rec_any(r)) {
        v = lane_id() == 0 ? lse_overlay<PsiT>(T, b) : 0.0;
        v = __shfl_sync(FULL, v, 0);
      } else {
        v = T.init_lse[0];
      }
    } else if (T.b_flags[b] & 1u) {
      v = T.init_lse[0];
    } else if constexpr (Exact) {
      v = 0.0;
      if (lane_id() == 0) v = lse_exact(reinterpret_cast<const double*>(psi) + (size_t)b * T.psi_stride,
                                        T.action_count, T.eta);
    } else {
      v = row_lse_fast<PsiT>(psi + (size_t)b * T.psi_stride, T.action_count, T.eta);
    }
    if (lane_id() == 0) T.b_lse[b] = v;
  }
}

// Fast mode: the CDF row of every dense PSI row from the belief's cached LSE (one warp per
// belief) -- after host-level edits and eta changes; a pass keeps them current itself.
template <class PsiT>
__global__ void k_dense_cdfs(vp_tree T) {
  const int nb = min(T.counters[0], T.cap_beliefs);
  const int warps = gridDim.x * (blockDim.x >> 5);
  const PsiT* psi = reinterpret_cast<const PsiT*>(T.psi);
  PsiT* cdf = reinterpret_cast<PsiT*>(T.psi_cdf);
  for (int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += warps) {
    const int r = dense_row_of<PsiT>(T, b);
    if (r >= 0)
      build_cdf_row<PsiT, false>(psi + (size_t)r * T.psi_stride, cdf + (size_t)r * T.psi_stride, T.action_count,
                                 T.eta, T.b_lse[b]);
  }
}

static int g_num_sms = 0;
static int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (!g_num_sms && cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    g_num_sms = 148;
  return g_num_sms;
}

__global__ void k_rehash(vp_tree T) {
  const int na = T.counters[VP_COUNTER_ACTIONS], nb = T.counters[0];
  const int total = na + nb;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    // ids below the extents that no node took (static per-row numbering) keep ckey ~0
    if (i < na) {
      if (T.a_ckey[i] == ~0ull) continue;
      const u64 key = ((u64)(u32)T.a_parent_belief[i] << 32) | (u32)T.a_action[i];
      put_final(slots(T.hash_a), T.hmask_a, key, (u32)i);
    } else {
      const int b = i - na;
      if (b == 0 || T.b_ckey[b] == ~0ull) continue;
      const u64 key = belief_key(T, T.b_parent_belief[b], T.b_parent_act[b], T.b_parent_action[b], T.b_parent_obs[b]);
      put_final(slots(T.hash_b), T.hmask_b, key, (u32)b);
    }
  }
}

// Root-state draw into work.states (hook / iterative path; vp_plan fuses it into k_search).
template <class Model>
__global__ void k_draw(vp_work W, const typename Model::State* particles, const double* cumw, int m, u64 key, int rk) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < W.n) reinterpret_cast<typename Model::State*>(W.states)[r] = draw_state(particles, cumw, m, key, r, rk);
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

// One search call: every warp carries 32 rows through all levels.
template <class Model, class PsiT, bool Exact, int RK>
__global__ void __launch_bounds__(kSearchWarps * 32) k_search(vp_tree T, vp_model M, vp_work W, vp_search_args S,
                                                              StageCfg sc, int rows) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) u64 s_bar[kSearchWarps];
  const int A = T.action_count;
  Stage<PsiT> sg = make_stage<PsiT>(smem_raw, s_bar, sc);
  // [stage rows | initial row (16-B padded) | initial CDF]
  PsiT* init_row = reinterpret_cast<PsiT*>(smem_raw) + (size_t)kSearchWarps * sc.rows * sc.stride;
  PsiT* init_cdf = init_row + T.psi_stride;
  for (int a = threadIdx.x; a < T.psi_stride; a += blockDim.x) {
    init_row[a] = a < A ? (PsiT)T.init_prefs[a] : (PsiT)0;
    if (a < A) init_cdf[a] = reinterpret_cast<const PsiT*>(T.init_cdf)[a];
  }
  typedef typename Model::State State;
  State* shared_state = nullptr;  // cooperative models: one record per warp, after the initial CDF
  if constexpr (coop_trait<Model>::value) {
    const size_t off = ((size_t)(init_cdf + A - reinterpret_cast<PsiT*>(smem_raw)) * sizeof(PsiT) + 15) / 16 * 16;
    shared_state = reinterpret_cast<State*>(smem_raw + off) + (threadIdx.x >> 5);
  }
  fence_async_smem();  // the initial row is the source of TMA bulk stores (lazy rows)
  // the leaf counter of the NEXT pass is reset here: its previous user (the
  // backup of the pass before this one) has finished
  if (blockIdx.x == 0 && threadIdx.x == 0) W.leaf_count[(S.pass + 1u) & 1u] = 0;
  __syncthreads();
  const int wi = blockIdx.x * kSearchWarps + (threadIdx.x >> 5);
  // node ids of this pass: extent + (level - depth0) n + row (read by every warp before the
  // last block advances the extents)
  const int base_b = T.counters[0], base_a = T.counters[VP_COUNTER_ACTIONS];
  if (wi * rows_per_search_warp<Model>(S.mode, rows) < W.n)
    search_warp<Model, PsiT, Exact, RK>(T, M, W, S, sg, init_cdf, init_row, wi, shared_state, rows, base_a, base_b);
  if (S.mode == VP_SEARCH_TRAJECTORY) return;  // creates no nodes
  // the last warp to finish advances the extents (every warp has used its base by then)
  __syncwarp();
  if (lane_id() == 0) {
    if (atomicAdd(&T.counters[VP_COUNTER_DONE], 1) == (int)(gridDim.x * kSearchWarps) - 1) {
      const long long span = (long long)W.n * (S.d_max - S.depth0);
      T.counters[0] = (int)min((long long)base_b + span, (long long)INT_MAX);
      T.counters[VP_COUNTER_ACTIONS] = (int)min((long long)base_a + span, (long long)INT_MAX);
      T.counters[VP_COUNTER_DONE] = 0;
    }
  }
}

template <class PsiT, bool Exact>
__global__ void __launch_bounds__(kBackupWarps * 32) k_backup(vp_tree T, vp_work W, u32 pass, double gamma, int rpw) {
  __shared__ double s_v[kBackupWarps][32];
  const int warp = threadIdx.x >> 5;
  const int wi = blockIdx.x * kBackupWarps + warp;
  if (wi * rpw >= W.leaf_count[pass & 1u]) return;
  backup_warp<PsiT, Exact>(T, W, pass, gamma, wi, s_v[warp], rpw);
}

template <class PsiT>
__global__ void __launch_bounds__(256) k_cdf_rows(vp_tree T, u32 pass) {
  cdf_rows_warp<PsiT>(T, pass);
}

template <class PsiT>
__global__ void k_root_argmax(vp_tree T, int* out) {
  warp_root_argmax<PsiT>(T, out);
}

// the planning step's result in one launch: the chosen action, then (live beliefs, live
// actions, overflow)
template <class PsiT>
__global__ void k_plan_result(vp_tree T, int* out) {
  warp_root_argmax<PsiT>(T, out);
  const int idx[3] = {VP_COUNTER_LIVE_B, VP_COUNTER_LIVE_A, 2};
  if (threadIdx.x < 3) out[1 + threadIdx.x] = T.counters[idx[threadIdx.x]];
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
enum KernelKind { KK_DRAW = 0, KK_SEARCH, KK_BACKUP, KK_TREE_INIT, KK_REHASH, KK_ARGMAX, KK_HOOK, KK_CDF, KK_COUNT };
static_assert(KK_COUNT == VP_KERNEL_KINDS, "kernel kinds out of sync with vpb200.h");
struct ProfRec {
  int kind;
  cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_prof_pool;
static size_t g_prof_used = 0;
static bool g_prof_on = false;
static std::atomic<long long> g_launches{0};

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
#ifndef VP_PLUGIN_ONLY  // a plug-in library instantiates its own model only (compile time)
    case VP_MODEL_MARS: return f(MarsModel());
    case VP_MODEL_TABULAR: return f(TabularModel());
    case VP_MODEL_SYNTHETIC: return f(SyntheticModel());
    case VP_MODEL_LIGHTDARK: return f(LightDarkModel());
    case VP_MODEL_NAVIGATION: return f(NavigationModel());
    case VP_MODEL_CROWDNAV: return f(CrowdNavModel());
#endif
#ifdef VP_PLUGIN_SOURCE
    case VP_MODEL_USER: return f(UserModel());
#endif
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

// One-time per-device settings (kernel shared-memory opt-in, stack limit) are
// applied on first use on EACH device and remembered per (device, what).
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
static size_t& device_setting(const void* what) {
  static std::map<std::pair<int, const void*>, size_t> done;
  return done[{current_device(), what}];
}
static bool ensure_smem_optin(const void* kernel, size_t bytes) {
  size_t& have = device_setting(kernel);
  if (bytes <= 48 * 1024 || bytes <= have) return true;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return false;
  have = bytes;
  return true;
}

// Per-thread stack for models whose records live in local memory (the one-lane
// CrowdNav step of the SIR / hook kernels): reserved before any launch or graph
// capture needs it.
static bool ensure_stack(size_t bytes) {
  static const char tag = 0;
  size_t& have = device_setting(&tag);
  if (have >= bytes) return true;
  size_t cur = 0;
  if (cudaDeviceGetLimit(&cur, cudaLimitStackSize) != cudaSuccess) return false;
  if (cur < bytes && cudaDeviceSetLimit(cudaLimitStackSize, bytes) != cudaSuccess) return false;
  have = bytes;
  return true;
}

template <class Model>
static bool state_size_ok(const vp_model& M) {
  if constexpr (std::is_same<Model, CrowdNavModel>::value) {
    if (M.crowd_people < 1 || M.crowd_people > kCrowdPeople || M.crowd_tracked < 0 ||
        M.crowd_tracked > kCrowdTracked || M.crowd_heur_len < 1 || !M.crowd_heur)
      return false;
    if (!ensure_stack(3 * sizeof(CrowdState))) return false;
  }
#ifdef VP_PLUGIN_SOURCE
  if constexpr (std::is_same<Model, UserModel>::value && coop_trait<Model>::value) {
    if (!ensure_stack(3 * sizeof(typename Model::State))) return false;
  }
#endif
#ifdef VP_PLUGIN_SOURCE
  if constexpr (std::is_same<Model, UserModel>::value) {
    if (!M.user_params || M.user_param_bytes < (int64_t)sizeof(UserModel::Params)) return false;
  }
#endif
  return M.state_bytes == (int)sizeof(typename Model::State);
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Leaves per backup warp.  The climbs of a warp's leaves are independent chains of
// dependent L2 round trips: when the pass is small, fewer leaves per warp (more
// warps per SM) hide more latency; when it fills the GPU anyway, full warps issue
// fewer instructions.  Sized for ~16 warps per SM of the 148, between 8 and 32
// (measured: C2 16k rows: 8 -> -7 % step time; C3 64k rows flat; C5 64k rows but
// deeper trees: 32, 16 costs +8 %).
// VP_LEAVES_PER_WARP overrides (measurement only).
// Rows per search warp (32; VP_ROWS_PER_WARP overrides, measurement only).
static int search_rows_per_warp(int) {
  static const int forced = env_int("VP_ROWS_PER_WARP", 0);
  return forced > 0 ? std::min(32, forced) : 32;
}

static int leaves_per_warp(int n) {
  static const int forced = env_int("VP_LEAVES_PER_WARP", 0);
  if (forced > 0) return std::min(32, forced);
  const int want = (n + 148 * 16 - 1) / (148 * 16);
  return want <= 8 ? 8 : want <= 16 ? 16 : 32;
}

// Staged-row geometry: rows padded to an odd number of 16-B chunks so the
// LDS.128 scans of 8 lanes in different rows hit different bank groups.
template <class PsiT>
static StageCfg stage_cfg(int A, int per_warp_bytes) {
  int chunks = (int)(((size_t)A * sizeof(PsiT) + 15) / 16);
  if ((chunks & 1) == 0) ++chunks;
  StageCfg c;
  c.stride = chunks * 16 / (int)sizeof(PsiT);
  c.rows = std::max(1, std::min(32, per_warp_bytes / (chunks * 16)));
  return c;
}

// Per-warp TMA stage budget.  Stage shared memory bounds the resident search
// warps; a pass wants all of its warps resident at once (one wave), so the
// budget shrinks as the warps per SM grow: 100 KB / warps-per-SM, 4-32 KB
// (measured: C2 512 warps -> 25 KB, 16-32 KB flat; C3 2048 warps -> 7 KB,
// 4-8 KB 11 % faster than 32 KB; C5's 64-B rows never fill it).
// VP_STAGE_KB overrides (measurement only).
static int stage_budget_bytes(int n, int rows_per_warp) {
  static const int forced = env_int("VP_STAGE_KB", 0);
  if (forced > 0) return forced * 1024;
  const int warps = (n + rows_per_warp - 1) / rows_per_warp;
  const int per_sm = std::max(1, (warps + num_sms() - 1) / num_sms());
  return std::min(32, std::max(4, 100 / per_sm)) * 1024;
}

// Search launch geometry: staged rows of every warp + the block's copies of
// the initial row and its CDF (+ one record per warp for cooperative models).
template <class Model, class PsiT, bool Exact>
static int32_t search_geometry(int A, int n, int mode, StageCfg& sc, size_t& smem) {
  const int rows = rows_per_search_warp<Model>(mode, search_rows_per_warp(n));
  sc = Exact ? StageCfg{0, 4} : stage_cfg<PsiT>(A, stage_budget_bytes(n, rows));
  const size_t padded = ((size_t)A * sizeof(PsiT) + 15) / 16 * 16 / sizeof(PsiT);
  smem = ((size_t)kSearchWarps * sc.rows * sc.stride + padded + (size_t)A) * sizeof(PsiT);
  if (coop_trait<Model>::value) smem = (smem + 15) / 16 * 16 + kSearchWarps * sizeof(typename Model::State);
  return VP_OK;
}

template <class Model, class PsiT, bool Exact>
static int32_t set_search_attr(size_t smem) {
  return ensure_smem_optin((const void*)k_search<Model, PsiT, Exact, VP_RNG_SPLITMIX64>, smem) &&
                 ensure_smem_optin((const void*)k_search<Model, PsiT, Exact, VP_RNG_PHILOX>, smem)
             ? VP_OK
             : VP_ERR_CUDA;
}

template <class Model, class PsiT, bool Exact>
static int32_t launch_search(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_search_args& S,
                             cudaStream_t st) {
  StageCfg sc;
  size_t smem;
  search_geometry<Model, PsiT, Exact>(T.action_count, W.n, S.mode, sc, smem);
  if (int32_t rc = set_search_attr<Model, PsiT, Exact>(smem)) return rc;
  const int rows = search_rows_per_warp(W.n);
  const int grid = blocks_for(blocks_for(W.n, rows_per_search_warp<Model>(S.mode, rows)), kSearchWarps);
  {
    Launch L_(KK_SEARCH, st);
    // the stream kind is a template constant: the reference's SplitMix64 path carries no Philox branch
    if (M.rng_kind == VP_RNG_PHILOX)
      k_search<Model, PsiT, Exact, VP_RNG_PHILOX><<<grid, kSearchWarps * 32, smem, st>>>(T, M, W, S, sc, rows);
    else
      k_search<Model, PsiT, Exact, VP_RNG_SPLITMIX64><<<grid, kSearchWarps * 32, smem, st>>>(T, M, W, S, sc, rows);
  }
  return check_launch();
}

template <class PsiT, bool Exact>
static int32_t launch_backup(const vp_tree& T, const vp_work& W, u32 pass, double gamma, cudaStream_t st) {
  const int rpw = leaves_per_warp(W.n);
  const int grid = blocks_for(blocks_for(W.n, rpw), kBackupWarps);
  {
    Launch L_(KK_BACKUP, st);
    k_backup<PsiT, Exact><<<grid, kBackupWarps * 32, 0, st>>>(T, W, pass, gamma, rpw);
  }
  if constexpr (!Exact) {  // the CDFs of the dense rows this backup changed
    Launch L_(KK_CDF, st);
    k_cdf_rows<PsiT><<<num_sms() * 4, 256, 0, st>>>(T, pass);
  }
  return check_launch();
}

// ---- whole planning step

template <class Model>
static int32_t enqueue_inputs(const vp_tree& T, const vp_work& W, const vp_plan_args& P, cudaStream_t st) {
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
  if (cudaMemsetAsync(W.leaf_count, 0, 2 * sizeof(int32_t), st) != cudaSuccess) return VP_ERR_CUDA;
  return VP_OK;
}

template <class PsiT, bool Exact>
static int32_t enqueue_tree_reset(const vp_tree& T, cudaStream_t st) {
  { Launch L_(KK_TREE_INIT, st); k_clear<<<num_sms() * 4, 256, 0, st>>>(T); }
  { Launch L_(KK_TREE_INIT, st); k_tree_init<PsiT, Exact><<<1, 256, 0, st>>>(T); }
  return check_launch();
}

// The launches of one fixed-iteration planning step.
template <class Model, class PsiT, bool Exact>
static int32_t enqueue_plan_kernels(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_plan_args& P,
                                    cudaStream_t st) {
  if (int32_t rc = enqueue_inputs<Model>(T, W, P, st)) return rc;
  if (int32_t rc = enqueue_tree_reset<PsiT, Exact>(T, st)) return rc;
  int d = 1;
  for (int it = 0; it < P.iterations; ++it) {
    vp_search_args S;
    memset(&S, 0, sizeof(S));
    S.depth0 = 0;
    S.d_max = d;
    S.pass = (u32)it + 1u;  // the tree is fresh: passes restart at 1
    S.search_key_dev = P.keys_dev + 2 * it + 1;
    S.particles = P.particles_dev;
    S.cum_weights = P.cumw_dev;
    S.draw_key_dev = P.keys_dev + 2 * it;
    S.m = P.m;
    if (int32_t rc = launch_search<Model, PsiT, Exact>(T, M, W, S, st)) return rc;
    if (int32_t rc = launch_backup<PsiT, Exact>(T, W, S.pass, P.gamma, st)) return rc;
    d = std::min(d + 1, P.d_max_cap);
  }
  { Launch L_(KK_ARGMAX, st); k_plan_result<PsiT><<<1, 32, 0, st>>>(T, P.out_dev); }
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
// Graph cache and capture streams are shared by every caller thread (ctypes releases the GIL):
// guarded by one mutex; one capture stream per device, and the device is part of the key.
static std::vector<GraphEntry> g_graphs;
static unsigned long long g_graph_clock = 0;
static std::map<int, cudaStream_t> g_capture_streams;
static std::mutex g_graph_mu;

template <class T>
static void append_pod(std::vector<unsigned char>& v, const T& x) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(&x);
  v.insert(v.end(), p, p + sizeof(T));
}

// mode 0: direct launches; 1: captured into a CUDA graph (replayed while
// pointers / sizes / model are unchanged).
template <class Model, class PsiT, bool Exact>
static int32_t run_plan(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_plan_args& P,
                        cudaStream_t st) {
  {
    StageCfg sc;
    size_t smem;
    search_geometry<Model, PsiT, Exact>(T.action_count, W.n, VP_SEARCH_FUSED, sc, smem);
    if (int32_t rc = set_search_attr<Model, PsiT, Exact>(smem)) return rc;
  }
  if (P.mode == 0 || g_prof_on) return enqueue_plan_kernels<Model, PsiT, Exact>(T, M, W, P, st);
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_graph_mu);
  std::vector<unsigned char> key;
  append_pod(key, dev);
  append_pod(key, T);
  append_pod(key, M);
  append_pod(key, W);
  append_pod(key, P);
  const int budget = stage_budget_bytes(W.n, 32);
  append_pod(key, budget);
  GraphEntry* hit = nullptr;
  for (auto& e : g_graphs)
    if (e.key == key) hit = &e;
  if (!hit) {
    cudaStream_t& g_capture_stream = g_capture_streams[dev];
    if (!g_capture_stream && cudaStreamCreateWithFlags(&g_capture_stream, cudaStreamNonBlocking) != cudaSuccess)
      return VP_ERR_CUDA;
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, st);
    cudaStreamWaitEvent(g_capture_stream, ev, 0);
    cudaEventDestroy(ev);
    cudaStreamSynchronize(g_capture_stream);
    const long long l0 = g_launches.load();
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

// ---- SIR belief update (belief.py:47-102)

template <class Model>
__global__ void k_sir_propagate(vp_model M, const typename Model::State* in, const double* w, int m, int a, u32 obs,
                                u64 key, typename Model::State* out, double* logw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  typename Model::State st = in[i];
  u32 o;
  double r;
  Model::step(M, st, a, key, (u64)i, o, r, M.rng_kind);  // step_batch(states, actions, rng.derive(retry).bind(rows))
  out[i] = st;
  logw[i] = log(w[i]) + Model::obs_loglik(M, st, a, obs);  // log(weights) + log_lik (belief.py:88-90)
}

// Cooperative models (CrowdNav): one warp per particle, the record staged in
// shared memory and stepped by Model::step_warp (bit-identical to step()).
constexpr int kCoopSirWarps = 4;

template <class Model>
__global__ void __launch_bounds__(kCoopSirWarps * 32) k_sir_propagate_coop(vp_model M, const typename Model::State* in,
                                                                            const double* w, int m, int a, u32 obs,
                                                                            u64 key, typename Model::State* out,
                                                                            double* logw) {
  typedef typename Model::State State;
  __shared__ State s_state[kCoopSirWarps];
  const int warp = threadIdx.x >> 5;
  const int i = blockIdx.x * kCoopSirWarps + warp;
  if (i >= m) return;
  State& st = s_state[warp];
  warp_copy_state(st, in[i]);
  u32 o;
  double r;
  Model::step_warp(M, st, a, key, (u64)i, true, o, r, M.rng_kind);
  warp_copy_state(out[i], st);
  if (lane_id() == 0) logw[i] = log(w[i]) + Model::obs_loglik(M, st, a, obs);
}

// One block: max over finite log-weights, shifted = exp(lw - max), its numpy
// pairwise sum, then the sequential cumsum of shifted / sum with cum[-1] = 1
// (belief.py:91-93, 50-52).  The two serial sums run on one thread in numpy
// order; everything else is block-parallel.  Up to kSirSmem particles the
// values live in shared memory, so the serial chains wait on shared-memory
// loads (fetched 8 ahead), not on L2 round trips.
constexpr int kSirSmem = 16384;

__global__ void k_sir_normalise(const double* logw, int m, double* cum, int* finite) {
  extern __shared__ double s_w[];
  __shared__ double s_max[32];
  __shared__ double s_total;
  double* w = m <= kSirSmem ? s_w : cum;
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double v = logw[i];
    if (v > -INFINITY) mx = fmax(mx, v);
  }
  mx = warp_max(mx);
  if (lane_id() == 0) s_max[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? s_max[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) s_max[0] = v;
  }
  __syncthreads();
  mx = s_max[0];
  if (mx == -INFINITY) {
    if (threadIdx.x == 0) finite[0] = 0;
    return;
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) w[i] = exp(logw[i] - mx);
  __syncthreads();
  if (threadIdx.x == 0) s_total = pairwise_sum([&](int i) -> double { return w[i]; }, 0, m);
  __syncthreads();
  const double total = s_total;
  for (int i = threadIdx.x; i < m; i += blockDim.x) w[i] = w[i] / total;  // numpy's vectorised divide
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    int i = 0;
    for (; i + 8 <= m; i += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = w[i + k];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc = (i + k) ? acc + v[k] : v[k];
        w[i + k] = acc;
      }
    }
    for (; i < m; ++i) {
      acc = i ? acc + w[i] : w[i];
      w[i] = acc;
    }
    finite[0] = 1;
  }
  __syncthreads();
  if (w != cum) {
    for (int i = threadIdx.x; i < m; i += blockDim.x) cum[i] = i == m - 1 ? 1.0 : w[i];
  } else if (threadIdx.x == 0) {
    cum[m - 1] = 1.0;
  }
}

// Fast-mode normaliser (fp32 closed loops): the same max / exp / divide, but the sum and the
// cumsum are one block-wide scan -- thread t owns the contiguous chunk [t C, t C + C) -- instead
// of numpy's serial order, so the CDF differs from numpy's by a few ulps and a resampled index
// can move only where (j + u0) / m falls within those ulps of a CDF edge.
__global__ void __launch_bounds__(1024) k_sir_normalise_fast(const double* logw, int m, double* cum, int* finite) {
  __shared__ double s_red[32];
  const int t = threadIdx.x, nt = blockDim.x, lane = lane_id(), warp = t >> 5;
  double mx = -INFINITY;
  for (int i = t; i < m; i += nt) {
    const double v = logw[i];
    if (v > -INFINITY) mx = fmax(mx, v);
  }
  mx = warp_max(mx);
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  mx = s_red[lane < (nt >> 5) ? lane : 0];
  mx = warp_max(mx);
  __syncthreads();
  if (mx == -INFINITY) {
    if (t == 0) finite[0] = 0;
    return;
  }
  const int C = (m + nt - 1) / nt;
  const int lo = min(m, t * C), hi = min(m, lo + C);
  double loc = 0.0;
  for (int i = lo; i < hi; ++i) {
    const double e = exp(logw[i] - mx);
    cum[i] = e;
    loc += e;
  }
  // block exclusive scan of the chunk sums
  const double incl = warp_inclusive_scan(loc);
  if (lane == 31) s_red[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const double v = lane < (nt >> 5) ? s_red[lane] : 0.0;
    s_red[lane] = warp_inclusive_scan(v);
  }
  __syncthreads();
  const double total = s_red[(nt >> 5) - 1];
  double run = incl - loc + (warp ? s_red[warp - 1] : 0.0);
  const double inv = 1.0 / total;
  for (int i = lo; i < hi; ++i) {
    run += cum[i];
    cum[i] = i == m - 1 ? 1.0 : run * inv;
  }
  if (t == 0) finite[0] = 1;
}

template <class Model>
__global__ void k_sir_resample(const typename Model::State* prop, const double* cum, int m, double u0,
                               typename Model::State* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const double pos = ((double)j + u0) / (double)m;
  int lo = 0, hi = m;  // searchsorted(cum, pos, side="right")
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cum[mid] > pos) hi = mid;
    else lo = mid + 1;
  }
  out[j] = prop[lo < m ? lo : m - 1];
}

// ---- latency probe (bench.py's latency roofline): one thread chases a random cycle of 128-B lines
// with dependent gpu-scope loads (L2: never an L1 hit) or dependent atomics (atom.add 0 returns
// the next pointer), timed with %globaltimer (ns) and clock64 (SM cycles).
__global__ void k_probe_chase(const u64* next, int hops, int atomic, u64 start, double* out) {
  u64 p = start;
  long long c0 = clock64();
  u64 t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < hops; ++i) {
    if (atomic) p = atomicAdd(const_cast<unsigned long long*>(next + p), 0ull);
    else p = ld_relaxed_u64(next + p);
  }
  u64 t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  const long long c1 = clock64();
  out[0] = (double)(t1 - t0) / hops;
  out[1] = (double)(c1 - c0) / hops;
  out[2] = (double)p;  // keeps the chain live
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
// draws of either stream kind (rk); normal != 0: Box-Muller normals
__global__ void k_rng_draws(u64 key, const int64_t* rows, int64_t n, int k, int rk, int normal, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 r = (u64)rows[i];
  if (k <= 0) out[i] = normal ? normal_j(key, r, 0, rk) : uniform1(key, r, rk);
  else
    for (int j = 1; j <= k; ++j)
      out[i * k + (j - 1)] = normal ? normal_j(key, r, (u64)j, rk) : uniform_j(key, r, (u64)j, rk);
}
__global__ void k_philox_blocks(const uint4* ctr, const uint2* key, int64_t n, uint4* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = philox4x32_10(ctr[i], key[i]);
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
  Model::step(M, s, act[i], key, (u64)rows[i], o, r, M.rng_kind);
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
template <class Model>
__global__ void k_model_loglik(vp_model M, const typename Model::State* st, int n, int a, u32 o, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = Model::obs_loglik(M, st[i], a, o);
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

// The PSI layout the kernels are compiled for: parity mode keeps one row per belief,
// fast mode dense rows for the busy beliefs plus overlay records.
static bool tree_ok(const vp_tree& T) {
  return T.action_count >= 1 && T.action_count < 65535 && T.b_rec && T.b_nact && T.a_slot && T.cap_dense >= 1 &&
         T.overlay_slots == (T.exact ? 0 : VP_OVERLAY_SLOTS) && (!T.exact || T.cap_dense >= T.cap_beliefs);
}

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

int64_t vp_launch_count(void) { return g_launches.load(); }

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
                       (int32_t)offsetof(vp_tree, init_cdf),
                       (int32_t)offsetof(vp_tree, a_ckey),
                       (int32_t)offsetof(vp_search_args, m),
                       (int32_t)offsetof(vp_model, mars_gpow),
                       (int32_t)offsetof(vp_tree, psi_cdf),
                       (int32_t)offsetof(vp_model, nav_log_miss), (int32_t)offsetof(vp_model, crowd_heur),
                       (int32_t)sizeof(CrowdState), (int32_t)offsetof(vp_tree, b_rec),
                       (int32_t)offsetof(vp_tree, a_slot), (int32_t)offsetof(vp_tree, cap_dense),
                       (int32_t)offsetof(vp_model, rng_kind), (int32_t)offsetof(vp_model, user_params),
                       (int32_t)offsetof(vp_model, user_param_bytes)};
  const int32_t m = (int32_t)(sizeof(v) / sizeof(v[0]));
  if (!out) return m;
  for (int32_t i = 0; i < n && i < m; ++i) out[i] = v[i];
  return m;
}

int32_t vp_tree_init(const vp_tree* t, void* stream) {
  if (!t || !tree_ok(*t)) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(t->hash_a, 0xff, (t->hmask_a + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  if (cudaMemsetAsync(t->hash_b, 0xff, (t->hmask_b + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  const vp_tree T = *t;
  return dispatch_psi(T.psi_dtype, T.exact, [&](auto z, auto ex) -> int32_t {
    return enqueue_tree_reset<decltype(z), decltype(ex)::value>(T, st);
  });
}

int32_t vp_tree_set_eta(const vp_tree* t, void* stream) {
  if (!t || !(t->eta > 0.0) || t->action_count < 1) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_tree T = *t;
  return dispatch_psi(T.psi_dtype, T.exact, [&](auto z, auto ex) -> int32_t {
    typedef decltype(z) PsiT;
    constexpr bool E = decltype(ex)::value;
    { Launch L_(KK_TREE_INIT, st); k_eta_init_row<PsiT, E><<<1, 32, 0, st>>>(T); }
    { Launch L_(KK_TREE_INIT, st); k_eta_rows<PsiT, E><<<num_sms() * 8, 256, 0, st>>>(T); }
    if (!E) { Launch L_(KK_TREE_INIT, st); k_dense_cdfs<PsiT><<<num_sms() * 8, 256, 0, st>>>(T); }
    return check_launch();
  });
}

int32_t vp_tree_build_cdfs(const vp_tree* t, void* stream) {
  if (!t || t->action_count < 1) return VP_ERR_INVALID;
  if (t->exact) return VP_OK;  // parity mode samples its PSI rows directly
  cudaStream_t st = (cudaStream_t)stream;
  const vp_tree T = *t;
  return dispatch_psi(T.psi_dtype, 0, [&](auto z, auto) -> int32_t {
    { Launch L_(KK_TREE_INIT, st); k_dense_cdfs<decltype(z)><<<num_sms() * 8, 256, 0, st>>>(T); }
    return check_launch();
  });
}

int32_t vp_tree_rehash(const vp_tree* t, void* stream) {
  if (!t) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(t->hash_a, 0xff, (t->hmask_a + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  if (cudaMemsetAsync(t->hash_b, 0xff, (t->hmask_b + 1) * sizeof(Slot), st) != cudaSuccess) return VP_ERR_CUDA;
  { Launch L_(KK_REHASH, st); k_rehash<<<num_sms() * 8, 256, 0, st>>>(*t); }
  return check_launch();
}

int32_t vp_tree_counts(const vp_tree* t, int32_t* host_out, void* stream) {
  if (!t || !host_out) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const int idx[5] = {VP_COUNTER_LIVE_B, VP_COUNTER_LIVE_A, 2, 0, VP_COUNTER_ACTIONS};
  for (int k = 0; k < 5; ++k)
    if (cudaMemcpyAsync(host_out + k, t->counters + idx[k], sizeof(int32_t), cudaMemcpyDeviceToHost, st) !=
        cudaSuccess)
      return VP_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return VP_ERR_CUDA;
  return VP_OK;
}

static bool work_ok(const vp_work& W) { return W.n >= 1 && W.n < (1 << 24) && W.max_levels >= 1 && W.max_levels <= 255; }

int32_t vp_draw_root_states(const vp_model* m, const vp_work* w, const void* particles, const double* cumw,
                            int32_t count, uint64_t key, void* stream) {
  if (!m || !w || !particles || !cumw || count < 1 || !work_ok(*w)) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_work W = *w;
  return dispatch_model(m->kind, [&](auto mdl) -> int32_t {
    typedef decltype(mdl) Model;
    if (!state_size_ok<Model>(*m)) return VP_ERR_INVALID;
    Launch L_(KK_DRAW, st);
    k_draw<Model><<<blocks_for(W.n, 256), 256, 0, st>>>(
        W, reinterpret_cast<const typename Model::State*>(particles), cumw, count, key, m->rng_kind);
    return check_launch();
  });
}

int32_t vp_search(const vp_tree* t, const vp_model* m, const vp_work* w, const vp_search_args* a, void* stream) {
  if (!t || !m || !w || !a || !work_ok(*w)) return VP_ERR_INVALID;
  if (!tree_ok(*t)) return VP_ERR_INVALID;
  if (a->depth0 < 0 || a->d_max < a->depth0 || a->d_max > w->max_levels || a->pass < 1) return VP_ERR_INVALID;
  if (a->particles && (!a->cum_weights || a->m < 1)) return VP_ERR_INVALID;
  if (a->mode < VP_SEARCH_FUSED || a->mode > VP_SEARCH_INSERT || a->row0 < 0) return VP_ERR_INVALID;
  if (a->mode == VP_SEARCH_TRAJECTORY &&
      (a->depth0 != 0 || a->start_beliefs || !w->trace_action || !w->trace_obs || !w->trace_reward))
    return VP_ERR_INVALID;
  if (a->mode == VP_SEARCH_INSERT && (!a->inject_actions || !a->inject_obs || !a->inject_reward || !a->inject_leaf))
    return VP_ERR_INVALID;
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
      return launch_search<Model, decltype(z), decltype(ex)::value>(T, M, W, S, st);
    });
  });
}

int32_t vp_plan(const vp_tree* t, const vp_model* m, const vp_work* w, const vp_plan_args* p, void* stream) {
  if (!t || !m || !w || !p || !work_ok(*w)) return VP_ERR_INVALID;
  if (!tree_ok(*t)) return VP_ERR_INVALID;
  if (p->iterations < 1 || p->d_max_cap < 1 || p->m < 1 || !p->keys_dev || !p->particles_dev || !p->cumw_dev ||
      !p->out_dev || (p->mode != 0 && p->mode != 1))
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

int32_t vp_backup(const vp_tree* t, const vp_work* w, uint32_t pass, double gamma, void* stream) {
  if (!t || !w || !work_ok(*w) || pass < 1) return VP_ERR_INVALID;
  if (!tree_ok(*t)) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_tree T = *t;
  const vp_work W = *w;
  return dispatch_psi(T.psi_dtype, T.exact, [&](auto z, auto ex) -> int32_t {
    return launch_backup<decltype(z), decltype(ex)::value>(T, W, pass, gamma, st);
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

int32_t vp_sir_weigh(const vp_model* mdl, const void* states, const double* weights, int32_t m, int32_t action,
                     uint32_t observation, uint64_t key, void* states_out, double* logw, double* cum, int32_t* finite,
                     int32_t exact, void* stream) {
  if (!mdl || !states || !weights || m < 1 || !states_out || !logw || !cum || !finite) return VP_ERR_INVALID;
  if (action < 0 || action >= mdl->action_count || observation > (uint32_t)mdl->obs_arity) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_model M = *mdl;
  return dispatch_model(M.kind, [&](auto md) -> int32_t {
    typedef decltype(md) Model;
    typedef typename Model::State State;
    if (!state_size_ok<Model>(M)) return VP_ERR_INVALID;
    {
      Launch L_(KK_HOOK, st);
      if constexpr (coop_trait<Model>::value)
        k_sir_propagate_coop<Model><<<blocks_for(m, kCoopSirWarps), kCoopSirWarps * 32, 0, st>>>(
            M, reinterpret_cast<const State*>(states), weights, m, action, observation, key,
            reinterpret_cast<State*>(states_out), logw);
      else
        k_sir_propagate<Model><<<blocks_for(m, 256), 256, 0, st>>>(M, reinterpret_cast<const State*>(states), weights,
                                                                     m, action, observation, key,
                                                                     reinterpret_cast<State*>(states_out), logw);
    }
    if (exact) {
      const size_t smem = m <= kSirSmem ? (size_t)m * sizeof(double) : 0;
      if (!ensure_smem_optin((const void*)k_sir_normalise, kSirSmem * sizeof(double))) return VP_ERR_CUDA;
      Launch L_(KK_HOOK, st);
      k_sir_normalise<<<1, 1024, smem, st>>>(logw, m, cum, finite);
    } else {
      Launch L_(KK_HOOK, st);
      k_sir_normalise_fast<<<1, 1024, 0, st>>>(logw, m, cum, finite);
    }
    return check_launch();
  });
}

int32_t vp_sir_resample(const vp_model* mdl, const void* prop, const double* cum, int32_t m, double u0,
                        void* states_out, void* stream) {
  if (!mdl || !prop || !cum || m < 1 || !states_out || !(u0 >= 0.0 && u0 < 1.0)) return VP_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_model M = *mdl;
  return dispatch_model(M.kind, [&](auto md) -> int32_t {
    typedef decltype(md) Model;
    typedef typename Model::State State;
    if (!state_size_ok<Model>(M)) return VP_ERR_INVALID;
    Launch L_(KK_HOOK, st);
    k_sir_resample<Model><<<blocks_for(m, 256), 256, 0, st>>>(reinterpret_cast<const State*>(prop), cum, m, u0,
                                                              reinterpret_cast<State*>(states_out));
    return check_launch();
  });
}

// Host-level tree mutation (tree.py:180-256 append_actions / append_beliefs):
// one thread per edge, the search's claim / numbering / creation-key protocol,
// so new nodes take reference ids n + rank in first-occurrence order at export.
}  // extern "C"

namespace vp {
template <class PsiT>
__global__ void k_append_actions(vp_tree T, const int32_t* beliefs, const int32_t* actions, const double* rewards,
                                 int n, u32 pass, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Slot* ha = slots(T.hash_a);
  const int b = beliefs[i], a = actions[i];
  const Claim cl = claim_key(ha, T.hmask_a, ((u64)(u32)b << 32) | (u32)a);
  int x;
  if (cl.won) {
    x = atomicAdd(&T.counters[VP_COUNTER_ACTIONS], 1);
    red_add(&T.counters[VP_COUNTER_LIVE_A], 1);
    if (x < T.cap_actions) {
      T.a_parent_belief[x] = b;
      T.a_action[x] = a;
      red_min(&T.a_ckey[x], creation_key(pass, 0, i));
      const int k = atomicAdd(&T.b_nact[b], 1);  // overlay slot (the search's protocol)
      T.a_slot[x] = k;
      if (T.overlay_slots && k == kOverlay) {
        const Rec<PsiT> r = load_rec<PsiT, true>(T, b);
        if (!r.dense_pass) materialise_dense<PsiT>(T, nullptr, b, r, nullptr, pass);
      }
    } else {
      T.counters[2] = 1;
    }
    publish(ha, cl.slot, (u32)x, pass);
  } else {
    const u64 w = wait_published(ha, cl.slot, cl.word);
    x = (int)(u32)w;
    if ((u32)(w >> 32) == pass && x < T.cap_actions) red_min(&T.a_ckey[x], creation_key(pass, 0, i));
  }
  if (x < T.cap_actions) {
    red_add(&T.a_reward[x], rewards[i]);  // np.add.at(reward, idx, r) (tree.py:216-217)
    red_add(&T.a_visits[x], 1);
  }
  out[i] = x < T.cap_actions ? x : -1;
}

}  // namespace vp

extern "C" {

__global__ void k_append_beliefs(vp_tree T, const int32_t* anodes, const uint32_t* obs, int n, u32 pass, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Slot* hb = slots(T.hash_b);
  const int x = anodes[i];
  const u32 o = obs[i];
  const Claim cl = claim_key(hb, T.hmask_b, belief_key(T, T.a_parent_belief[x], T.a_action[x], x, o));
  int c;
  if (cl.won) {
    c = atomicAdd(&T.counters[0], 1);
    red_add(&T.counters[VP_COUNTER_LIVE_B], 1);
    if (c < T.cap_beliefs) {
      const int pb = T.a_parent_belief[x];
      T.b_parent_action[c] = x;
      T.b_parent_obs[c] = o;
      T.b_parent_belief[c] = pb;
      T.b_parent_act[c] = T.a_action[x];
      T.b_depth[c] = T.b_depth[pb] + 1;  // tree.py:253
      T.b_lse[c] = T.init_lse[0];
      T.b_flags[c] = 3u;  // PSI row == init_prefs, not materialised (tree.py:253)
      red_min(&T.b_ckey[c], creation_key(pass, 0, i));
    } else {
      T.counters[2] = 1;
    }
    publish(hb, cl.slot, (u32)c, pass);
  } else {
    const u64 w = wait_published(hb, cl.slot, cl.word);
    c = (int)(u32)w;
    if ((u32)(w >> 32) == pass && c < T.cap_beliefs) red_min(&T.b_ckey[c], creation_key(pass, 0, i));
  }
  out[i] = c < T.cap_beliefs ? c : -1;
}

int32_t vp_tree_append_actions(const vp_tree* t, const int32_t* beliefs, const int32_t* actions, const double* rewards,
                               int32_t n, uint32_t pass, int32_t* out, void* stream) {
  if (!t || n < 0 || (n && (!beliefs || !actions || !rewards || !out)) || pass == 0) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  Launch L_(KK_HOOK, (cudaStream_t)stream);
  if (t->psi_dtype == VP_PSI_F32)
    k_append_actions<float><<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*t, beliefs, actions, rewards, n, pass,
                                                                                   out);
  else
    k_append_actions<double><<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*t, beliefs, actions, rewards, n,
                                                                                    pass, out);
  return check_launch();
}

int32_t vp_tree_append_beliefs(const vp_tree* t, const int32_t* action_nodes, const uint32_t* observations, int32_t n,
                               uint32_t pass, int32_t* out, void* stream) {
  if (!t || n < 0 || (n && (!action_nodes || !observations || !out)) || pass == 0) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  Launch L_(KK_HOOK, (cudaStream_t)stream);
  k_append_beliefs<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*t, action_nodes, observations, n, pass, out);
  return check_launch();
}

__global__ void k_broadcast_record(u64* rec, long long words_total, int words, const u64* src, int keep_lo,
                                   int keep_hi) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words_total;
       i += (long long)gridDim.x * blockDim.x) {
    const int w = (int)(i % words);
    if (w < keep_lo || w >= keep_hi) rec[i] = src[w];
  }
}

int32_t vp_plan_keys(uint64_t key, int32_t iterations, uint64_t* out) {
  if (iterations < 0 || (iterations && !out)) return VP_ERR_INVALID;
  for (int32_t i = 0; i < iterations; ++i) {
    const uint64_t it = fold(key, (uint64_t)i);
    out[2 * i] = fold(it, 0);      // SITE_DRAW
    out[2 * i + 1] = fold(it, 1);  // SITE_SEARCH
  }
  return VP_OK;
}

// Host packer of MARS particle records (the e2e path packs the caller's belief every planning
// step): 8 rock flags at a time turned into 8 bits by one multiply.
static inline uint64_t bytes8_to_bits(uint64_t v) {
  return ((v & 0x0101010101010101ull) * 0x0102040810204080ull) >> 56;
}

int32_t vp_pack_mars_states(const int64_t* x, const int64_t* y, const uint8_t* terminal, const uint8_t* rocks,
                            int64_t n, int32_t m, void* dst) {
  if (n < 0 || m < 0 || m > 64 || (n && (!x || !y || !terminal || !dst || (m && !rocks)))) return VP_ERR_INVALID;
  uint64_t* out = static_cast<uint64_t*>(dst);
  const int chunks = (m + 7) / 8;
  // rows whose whole-chunk reads stay inside the rocks array
  const int64_t total = n * (int64_t)m;
  const int64_t safe = m ? std::max<int64_t>(0, (total - 8 * chunks) / m) : n;
  const uint64_t mask = m >= 64 ? ~0ull : ((1ull << m) - 1ull);
  for (int64_t i = 0; i < n; ++i) {
    out[2 * i] = (uint64_t)(x[2 * i] & 0xff) | (uint64_t)(y[2 * i] & 0xff) << 8 |
                 (uint64_t)(x[2 * i + 1] & 0xff) << 16 | (uint64_t)(y[2 * i + 1] & 0xff) << 24 |
                 (uint64_t)(terminal[i] != 0) << 32;
    const uint8_t* r = rocks + i * (int64_t)m;
    uint64_t bits = 0;
    if (i < safe) {
      for (int c = 0; c < chunks; ++c) {
        uint64_t v;
        memcpy(&v, r + 8 * c, 8);
        bits |= bytes8_to_bits(v) << (8 * c);
      }
      bits &= mask;
    } else {
      for (int k = 0; k < m; ++k) bits |= (uint64_t)(r[k] != 0) << k;
    }
    out[2 * i + 1] = bits;
  }
  return VP_OK;
}

int32_t vp_broadcast_record(void* records, int32_t m, int32_t record_bytes, const void* source, int32_t keep_lo,
                            int32_t keep_hi, void* stream) {
  if (!records || !source || m < 1 || record_bytes < 8 || record_bytes % 8 || keep_lo % 8 || keep_hi % 8 ||
      keep_lo < 0 || keep_hi < keep_lo || keep_hi > record_bytes)
    return VP_ERR_INVALID;
  const long long total = (long long)m * (record_bytes / 8);
  Launch L_(KK_HOOK, (cudaStream_t)stream);
  k_broadcast_record<<<(int)std::min<long long>((total + 255) / 256, 148LL * 16), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<u64*>(records), total, record_bytes / 8, reinterpret_cast<const u64*>(source), keep_lo / 8,
      keep_hi / 8);
  return check_launch();
}

#ifdef VP_PHASE_CLOCKS
// measurement builds: read (and clear) the per-phase cycle sums of the search
int32_t vp_debug_phases(unsigned long long* host_out) {
  if (cudaMemcpyFromSymbol(host_out, vp::g_phase_cycles, 24 * sizeof(unsigned long long)) != cudaSuccess)
    return VP_ERR_CUDA;
  unsigned long long z[24] = {0};
  return cudaMemcpyToSymbol(vp::g_phase_cycles, z, sizeof(z)) == cudaSuccess ? VP_OK : VP_ERR_CUDA;
}
// the backup completion trace out (returns the entry count), then reset
int32_t vp_debug_trace(unsigned long long* host_out, int32_t max_n) {
  unsigned int n = 0;
  if (cudaMemcpyFromSymbol(&n, vp::g_trace_n, sizeof(n)) != cudaSuccess) return -1;
  n = std::min<unsigned int>(n, 1u << 21);
  if (host_out && n &&
      cudaMemcpyFromSymbol(host_out, vp::g_trace, sizeof(unsigned long long) * std::min<unsigned>(n, (unsigned)max_n)) !=
          cudaSuccess)
    return -1;
  const unsigned int z = 0;
  cudaMemcpyToSymbol(vp::g_trace_n, &z, sizeof(z));
  return (int32_t)n;
}
#endif

int32_t vp_probe_latency(const uint64_t* next, int32_t hops, int32_t atomic, uint64_t start, double* out,
                         void* stream) {
  if (!next || hops < 1 || !out) return VP_ERR_INVALID;
  k_probe_chase<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<const u64*>(next), hops, atomic, start, out);
  return check_launch();
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

int32_t vp_rng_draws(uint64_t key, const int64_t* rows, int64_t n, int32_t k, int32_t rng_kind, int32_t normal,
                     double* out, void* stream) {
  if (n < 0 || (n && (!rows || !out)) || (rng_kind != VP_RNG_SPLITMIX64 && rng_kind != VP_RNG_PHILOX))
    return VP_ERR_INVALID;
  if (!n) return VP_OK;
  k_rng_draws<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(key, rows, n, k, rng_kind, normal, out);
  return check_launch();
}

int32_t vp_philox4x32_10(const uint32_t* counters, const uint32_t* keys, int64_t n, uint32_t* out, void* stream) {
  if (n < 0 || (n && (!counters || !keys || !out))) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  k_philox_blocks<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uint4*>(counters), reinterpret_cast<const uint2*>(keys), n, reinterpret_cast<uint4*>(out));
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

int32_t vp_model_obs_loglik(const vp_model* m, const void* states, int32_t n, int32_t action, uint32_t observation,
                            double* out, void* stream) {
  if (!m || n < 0 || action < 0 || action >= m->action_count) return VP_ERR_INVALID;
  if (!n) return VP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const vp_model M = *m;
  return dispatch_model(M.kind, [&](auto mdl) -> int32_t {
    typedef decltype(mdl) Model;
    if (!state_size_ok<Model>(M)) return VP_ERR_INVALID;
    k_model_loglik<Model><<<blocks_for(n, 256), 256, 0, st>>>(
        M, reinterpret_cast<const typename Model::State*>(states), n, action, observation, out);
    return check_launch();
  });
}

int32_t vp_plugin_info(int32_t* state_bytes) {
#ifdef VP_PLUGIN_SOURCE
  if (state_bytes) *state_bytes = (int32_t)sizeof(UserModel::State);
  return 1;
#else
  if (state_bytes) *state_bytes = 0;
  return 0;
#endif
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
