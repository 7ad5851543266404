// vp_kernels.cu -- B200 (sm_100a) kernels of the PORPP planning step and the
// C ABI declared in include/vpb200.h.
//
// One search level (search.py:106-118) is four launches over the n rows:
//   K1 level_sample   : frontier belief -> softmax draw -> G(s,a) -> claim (b,a)
//   K2 assign_actions : first-occurrence scan -> new action ids (tree.py:180-218)
//   K3 accum_probe    : reward/visit accumulation, claim (anode, o)
//   K4 assign_beliefs : first-occurrence scan -> new belief rows (tree.py:220-256)
// The backup (backup.py:75-114) is one pass over the leaf list and two
// launches per level over the per-level distinct lists recorded by search:
//   Q / PSI scatter over the level's action nodes, LSE over its beliefs.
// Nothing here is a dense contraction: every kernel is HBM / latency bound.
//
// PSI rows are created lazily: a new belief only gets a "fresh" flag (its row
// equals the initial row); the sampler draws fresh beliefs from one shared
// initial CDF, and the backup materialises a row the first time it updates it.
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <cfloat>
#include <type_traits>
#include <algorithm>
#include <vector>

#include "vp_common.cuh"
#include "vp_models.cuh"

namespace vp {

static thread_local cudaError_t g_last_cuda = cudaSuccess;

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ Slot* slots(void* p) { return reinterpret_cast<Slot*>(p); }

// ------------------------------------------------------------------ exp helpers (fast mode)
// The fast sampler and the fast LSE evaluate exp(eta * psi - shift) as
// exp2(fma(eta*log2e, psi, -shift*log2e)); float uses ex2.approx, double exp2.
__device__ __forceinline__ float fexp2(float x) { return exp2f(x); }
__device__ __forceinline__ double fexp2(double x) { return exp2(x); }
__device__ __forceinline__ float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double ffma(double a, double b, double c) { return __fma_rn(a, b, c); }

// ------------------------------------------------------------------ LSE

// Fast LSE: warp per row, max then sum of exp (backup.py:34-41 formula).
template <class PsiT>
__device__ double warp_lse_fast(const PsiT* row, int A, double eta) {
  typedef PsiT CT;
  const int lane = lane_id();
  const CT e = (CT)eta;
  CT m = -(CT)INFINITY;
  for (int a = lane; a < A; a += 32) {
    const CT z = e * row[a];
    m = z > m ? z : m;
  }
  m = warp_max(m);
  const CT e2 = (CT)(eta * 1.4426950408889634), m2 = m * (CT)1.4426950408889634;
  CT s = 0;
  for (int a = lane; a < A; a += 32) s += fexp2(ffma(e2, row[a], -m2));
  s = warp_sum(s);
  return (double)m / eta + log((double)s) / eta;
}

// numpy-order LSE for the fp64 parity mode: m/eta + log(pairwise sum)/eta.
__device__ double lse_exact(const double* row, int A, double eta) {
  double m = -INFINITY;
  for (int a = 0; a < A; ++a) m = fmax(m, eta * row[a]);
  auto ex = [&](int a) -> double { return exp(eta * row[a] - m); };
  const double s = pairwise_sum(ex, 0, A);
  return m / eta + log(s) / eta;
}

// ------------------------------------------------------------------ categorical draws

// numpy-order inverse CDF draw (search.py:46-54 then 77-79, 83).
__device__ int sample_exact(const double* row, int A, double eta, double u) {
  double m = -INFINITY;
  for (int a = 0; a < A; ++a) m = fmax(m, eta * row[a]);
  auto ex = [&](int a) -> double { return exp(eta * row[a] - m); };
  const double s = pairwise_sum(ex, 0, A);
  double cum = 0.0;
  for (int a = 0; a < A; ++a) {
    const double p = ex(a) / s;
    cum = a ? cum + p : p;
    if (cum > u) return a;
  }
  return A - 1;
}

// Fast draw: the probabilities are exp(eta (psi - LSE)), normalised by the
// row's cached LSE, accumulated left to right until the running sum exceeds u
// (clamp |A|-1, search.py:83).  The scalar and the vectorised (staged shared
// memory) versions perform the identical floating-point sequence.
template <class CT>
__device__ __forceinline__ int scan_cdf_scalar(const CT* row, int A, CT e2, CT sh2, CT u) {
  CT cum = 0;
  for (int a = 0; a < A; ++a) {
    cum += fexp2(ffma(e2, row[a], -sh2));
    if (cum > u) return a;
  }
  return A - 1;
}
template <class CT>
struct Vec16;
template <>
struct Vec16<float> {
  typedef float4 T;
  static constexpr int N = 4;
  static __device__ __forceinline__ void get(const T& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
};
template <>
struct Vec16<double> {
  typedef double2 T;
  static constexpr int N = 2;
  static __device__ __forceinline__ void get(const T& v, double* o) { o[0] = v.x; o[1] = v.y; }
};
template <class CT>
__device__ __forceinline__ int scan_cdf_vec(const CT* row, int A, CT e2, CT sh2, CT u) {
  typedef Vec16<CT> V;
  CT cum = 0;
  const typename V::T* rv = reinterpret_cast<const typename V::T*>(row);
  for (int a0 = 0; a0 < A; a0 += V::N) {
    CT x[V::N];
    V::get(rv[a0 / V::N], x);
#pragma unroll
    for (int j = 0; j < V::N; ++j) {
      if (a0 + j < A) {
        cum += fexp2(ffma(e2, x[j], -sh2));
        if (cum > u) return a0 + j;
      }
    }
  }
  return A - 1;
}
// First index whose (initial-row) CDF value exceeds u.
template <class CT>
__device__ __forceinline__ int search_cdf(const CT* cdf, int A, CT u) {
  int lo = 0, hi = A;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cdf[mid] > u) hi = mid;
    else lo = mid + 1;
  }
  return lo < A ? lo : A - 1;
}

// ------------------------------------------------------------------ TMA bulk staging

__device__ __forceinline__ u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// ------------------------------------------------------------------ warp helpers

// Warp-aggregated probe/claim: lanes with equal keys elect their lowest lane
// (= smallest row, rows are contiguous per warp) to touch the table once.
__device__ __forceinline__ u32 warp_claim(Slot* tab, u64 mask, u64 key, u32 row, bool active) {
  const u32 grp = __match_any_sync(FULL, active ? key : kEmptyKey);
  const int leader = __ffs(grp) - 1;
  u32 word = 0;
  if (active && lane_id() == leader) {
    bool existing;
    u32 id;
    const u32 s = probe_claim(tab, mask, key, row, existing, id);
    word = s | (existing ? kExistBit : 0u);
  }
  return __shfl_sync(FULL, word, leader);
}

// Dedup into a per-level list via per-node stamps (one stamp per level).
__device__ __forceinline__ void warp_list_once(u32* stamp, int node, u32 value, bool active, int* count,
                                               int* list) {
  const u32 grp = __match_any_sync(FULL, active ? (u32)node : 0xffffffffu);
  const int leader = __ffs(grp) - 1;
  if (active && lane_id() == leader) {
    if (atomicExch(&stamp[node], value) != value) {
      const int pos = atomicAdd(count, 1);
      list[pos] = node;
    }
  }
}

// Write the initial PSI row into belief b if it is still lazily fresh.
template <class PsiT>
__device__ __forceinline__ void warp_materialise(const vp_tree& T, int b) {
  if (!(T.b_flags[b] & 1)) return;
  PsiT* row = reinterpret_cast<PsiT*>(T.psi) + (size_t)b * T.psi_stride;
  for (int a = lane_id(); a < T.action_count; a += 32) row[a] = (PsiT)T.init_prefs[a];
  __syncwarp();
  if (lane_id() == 0) T.b_flags[b] = 0;
}

// ------------------------------------------------------------------ tree init / rehash

template <class PsiT, bool Exact>
__global__ void k_tree_init(vp_tree T) {
  PsiT* psi = reinterpret_cast<PsiT*>(T.psi);
  const int A = T.action_count;
  for (int a = threadIdx.x; a < A; a += blockDim.x) psi[a] = (PsiT)T.init_prefs[a];
  __syncthreads();
  if (threadIdx.x < 32) {
    double v;
    if constexpr (Exact) {
      v = 0.0;
      if (threadIdx.x == 0) v = lse_exact(reinterpret_cast<const double*>(psi), A, T.eta);
    } else {
      v = warp_lse_fast<PsiT>(psi, A, T.eta);
    }
    if (threadIdx.x == 0) {
      T.init_lse[0] = v;
      T.b_lse[0] = v;
      // CDF of the initial row with the sampler's exact arithmetic
      PsiT* cdf = reinterpret_cast<PsiT*>(T.init_cdf);
      const PsiT e2 = (PsiT)(T.eta * 1.4426950408889634), sh2 = (PsiT)(T.eta * v * 1.4426950408889634);
      PsiT cum = 0;
      for (int a = 0; a < A; ++a) {
        cum += fexp2(ffma(e2, psi[a], -sh2));
        cdf[a] = cum;
      }
      T.b_parent_action[0] = -1;
      T.b_parent_obs[0] = 0xffffffffu;
      T.b_depth[0] = 0;
      T.b_value[0] = 0.0;
      T.b_weight[0] = 0.0;
      T.b_stamp[0] = 0;
      T.b_flags[0] = 0;
      T.counters[0] = 1;
      T.counters[1] = 0;
      T.counters[2] = 0;
    }
  }
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

// ------------------------------------------------------------------ root draw

template <class Model>
__global__ void k_draw(vp_work W, const typename Model::State* particles, const double* cumw, int m, u64 key,
                       const u64* key_dev) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= W.n) return;
  const double u = uniform1(key_dev ? *key_dev : key, (u64)r);
  int lo = 0, hi = m;  // first index with cum > u  (searchsorted side=right)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cumw[mid] > u) hi = mid;
    else lo = mid + 1;
  }
  const int idx = lo < m - 1 ? lo : m - 1;
  reinterpret_cast<typename Model::State*>(W.states)[r] = particles[idx];
}

// ------------------------------------------------------------------ K1 level_sample

struct StageCfg {
  int rows;     // G: PSI rows staged per warp per batch
  int stride;   // staged row stride in PsiT elements (odd multiple of 16 bytes)
};

// Frontier belief of row r at `level` (hash_b slot written by K3 of level-1).
__device__ __forceinline__ int frontier_of(const vp_tree& T, const vp_work& W, const vp_search_args& S, int level,
                                           int r) {
  if (level == S.depth0) return S.start_beliefs ? S.start_beliefs[r] : 0;
  const u32 sl = (u32)W.slot_b[r] & ~kExistBit;
  const int b = (int)slots(T.hash_b)[sl].id;
  if (W.trace_belief) W.trace_belief[(size_t)(level - 1) * W.n + r] = b;
  return b;
}

// Model step + claim of (b, a) in hash_a; shared tail of both K1 variants.
template <class Model>
__device__ __forceinline__ void step_and_claim(const vp_tree& T, const vp_model& M, const vp_work& W, int level,
                                               u64 lkey, int r, bool active, int b, int a) {
  const int n = W.n;
  u64 key = 0;
  if (active) {
    typename Model::State st = reinterpret_cast<typename Model::State*>(W.states)[r];
    u32 o;
    double rw;
    Model::step(M, st, a, fold(lkey, 1), (u64)r, o, rw);  // level_rng.derive(1) (search.py:113-115)
    reinterpret_cast<typename Model::State*>(W.states)[r] = st;
    W.obs[r] = o;
    W.reward[r] = rw;
    W.action[r] = a;
    if (W.trace_action) {
      W.trace_action[(size_t)level * n + r] = a;
      W.trace_obs[(size_t)level * n + r] = o;
    }
    key = ((u64)(u32)b << 32) | (u32)a;
  }
  const u32 word = warp_claim(slots(T.hash_a), T.hmask_a, key, (u32)r, active);
  if (active) W.slot_a[r] = (int)word;
}

// Fast mode (fp32 or fp64 PSI).  Rows of the warp whose belief is fresh draw
// from the shared initial CDF; the distinct non-fresh beliefs' PSI rows are
// staged into shared memory with TMA bulk copies (one cp.async.bulk per row,
// completion on a per-warp mbarrier), then every lane scans its own row.
template <class Model, class PsiT>
__global__ void __launch_bounds__(128) k_level_sample(vp_tree T, vp_model M, vp_work W, vp_search_args S, int level,
                                                      u32 stamp, StageCfg sc) {
  const u64 lkey = fold(S.search_key_dev ? *S.search_key_dev : S.search_key, (u64)level);  // search.py:107
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) u64 s_bar[4];
  const int n = W.n;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = r < n;
  const int A = T.action_count;
  if (blockIdx.x == 0 && threadIdx.x == 0) W.level_base[2 * level] = T.counters[1];
  u64* bar = &s_bar[warp];
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();

  const int b = active ? frontier_of(T, W, S, level, r) : 0;
  warp_list_once(T.b_stamp, b, stamp, active, &W.fcount[level], W.flist + (size_t)level * n);
  const double u = active ? uniform1(fold(lkey, 0), (u64)r) : 0.0;  // level_rng.derive(0) (search.py:110)

  int a = 0;
  if (S.inject_actions) {
    a = active ? S.inject_actions[(size_t)level * n + r] : 0;
  } else {
    const bool fresh = active && (T.b_flags[b] & 1);
    const bool need = active && !fresh;
    if (fresh) a = search_cdf(reinterpret_cast<const PsiT*>(T.init_cdf), A, (PsiT)u);
    const u32 grp = __match_any_sync(FULL, need ? (u32)b : 0xffffffffu);
    const int my_leader = __ffs(grp) - 1;
    const u32 leaders = __ballot_sync(FULL, need && lane == my_leader);
    const int K = __popc(leaders);
    const int my_slot = need ? __popc(leaders & ((1u << my_leader) - 1u)) : -1;
    const double lse = need ? T.b_lse[b] : 0.0;
    const PsiT e2 = (PsiT)(T.eta * 1.4426950408889634), sh2 = (PsiT)(T.eta * lse * 1.4426950408889634);
    PsiT* stage = reinterpret_cast<PsiT*>(smem_raw) + (size_t)warp * sc.rows * sc.stride;
    const PsiT* psi = reinterpret_cast<const PsiT*>(T.psi);
    const u32 row_bytes = (u32)(((size_t)A * sizeof(PsiT) + 15) & ~(size_t)15);
    u32 phase = 0;
    u32 pending = leaders;
    for (int s0 = 0; s0 < K; s0 += sc.rows) {
      const int cnt = min(sc.rows, K - s0);
      fence_async_smem();
      if (lane == 0) mbar_expect_tx(bar, row_bytes * (u32)cnt);
      __syncwarp();
      // the j-th pending leader copies its belief's row into stage slot j
      const bool copier = need && lane == my_leader && my_slot >= s0 && my_slot < s0 + cnt;
      if (copier) bulk_g2s(stage + (size_t)(my_slot - s0) * sc.stride, psi + (size_t)b * T.psi_stride, row_bytes,
                           bar);
      mbar_wait(bar, phase);
      phase ^= 1u;
      if (need && my_slot >= s0 && my_slot < s0 + cnt)
        a = scan_cdf_vec<PsiT>(stage + (size_t)(my_slot - s0) * sc.stride, A, e2, sh2, (PsiT)u);
      __syncwarp();
    }
    (void)pending;
  }
  step_and_claim<Model>(T, M, W, level, lkey, r, active, b, a);
}

// fp64 parity mode: thread per row, numpy operation order, no staging.
template <class Model>
__global__ void __launch_bounds__(128) k_level_sample_exact(vp_tree T, vp_model M, vp_work W, vp_search_args S,
                                                            int level, u32 stamp) {
  const u64 lkey = fold(S.search_key_dev ? *S.search_key_dev : S.search_key, (u64)level);
  const int n = W.n;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = r < n;
  const int A = T.action_count;
  if (blockIdx.x == 0 && threadIdx.x == 0) W.level_base[2 * level] = T.counters[1];
  const int b = active ? frontier_of(T, W, S, level, r) : 0;
  warp_list_once(T.b_stamp, b, stamp, active, &W.fcount[level], W.flist + (size_t)level * n);
  const double u = active ? uniform1(fold(lkey, 0), (u64)r) : 0.0;
  int a = 0;
  if (active) {
    if (S.inject_actions) {
      a = S.inject_actions[(size_t)level * n + r];
    } else {
      const double* row = (T.b_flags[b] & 1) ? T.init_prefs
                                             : reinterpret_cast<const double*>(T.psi) + (size_t)b * T.psi_stride;
      a = sample_exact(row, A, T.eta, u);
    }
  }
  step_and_claim<Model>(T, M, W, level, lkey, r, active, b, a);
}

// ------------------------------------------------------------------ K2/K4 first-occurrence scans

// Number the rows that won their key this level, in row order (one row per
// thread, one tile per block, tiles chained by decoupled look-back), and
// write the new nodes' columns.  WhichTable: 0 = actions, 1 = beliefs.
template <int WhichTable>
__global__ void __launch_bounds__(VP_SCAN_TILE) k_assign(vp_tree T, vp_work W, int level, u32 epoch) {
  __shared__ u32 s_tile;
  __shared__ u32 s_warp[VP_SCAN_TILE / 32];
  __shared__ u32 s_excl;
  constexpr int NW = VP_SCAN_TILE / 32;
  const int n = W.n;
  Slot* tab = slots(WhichTable ? T.hash_b : T.hash_a);
  const int* slot_of = WhichTable ? W.slot_b : W.slot_a;
  if (threadIdx.x == 0) s_tile = atomicAdd(&W.scan_ticket[0], 1u);
  __syncthreads();
  const int tile = (int)s_tile;
  const int r = tile * VP_SCAN_TILE + threadIdx.x;
  u32 sl = 0;
  bool win = false;
  if (r < n) {
    const u32 w = (u32)slot_of[r];
    sl = w & ~kExistBit;
    if (!(w & kExistBit)) win = ld_volatile_u32(&tab[sl].id) == (kPending | (u32)r);
  }
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const u32 ballot = __ballot_sync(FULL, win);
  const u32 below = __popc(ballot & ((1u << lane) - 1u));
  if (lane == 0) s_warp[warp] = __popc(ballot);
  __syncthreads();
  if (warp == 0) {
    const u32 v = lane < NW ? s_warp[lane] : 0;
    const u32 vi = warp_inclusive_scan(v);
    if (lane < NW) s_warp[lane] = vi - v;
    const u32 agg = __shfl_sync(FULL, vi, NW - 1);
    const u32 excl = tile_lookback_warp(reinterpret_cast<u64*>(W.scan_status), tile, agg, epoch);
    if (lane == 0) {
      s_excl = excl;
      const int ntiles = (n + VP_SCAN_TILE - 1) / VP_SCAN_TILE;
      if (tile == ntiles - 1) {
        const int base = W.level_base[2 * level + WhichTable];
        T.counters[WhichTable ? 0 : 1] = base + (int)(excl + agg);
        W.scan_ticket[0] = 0;
      }
    }
  }
  __syncthreads();
  if (!win) return;
  const int id = W.level_base[2 * level + WhichTable] + (int)(s_excl + s_warp[warp] + below);
  Slot& s = tab[sl];
  s.id = (u32)id;
  const int cap = WhichTable ? T.cap_beliefs : T.cap_actions;
  if (id >= cap) {
    T.counters[2] = 1;  // overflow: the host fails the plan loudly
    return;
  }
  const u64 key = s.key;
  if (WhichTable == 0) {
    T.a_parent_belief[id] = (int)(key >> 32);
    T.a_action[id] = (int)(u32)key;
    T.a_reward[id] = 0.0;
    T.a_visits[id] = 0;
    T.a_num[id] = 0.0;
    T.a_den[id] = 0.0;
    T.a_stamp[id] = 0;
  } else {
    const int pa = (int)(key >> 32);
    T.b_parent_action[id] = pa;
    T.b_parent_obs[id] = (u32)key;
    T.b_depth[id] = T.b_depth[T.a_parent_belief[pa]] + 1;
    T.b_lse[id] = T.init_lse[0];
    T.b_value[id] = 0.0;
    T.b_weight[id] = 0.0;
    T.b_stamp[id] = 0;
    T.b_flags[id] = 1;  // PSI row lazily equal to the initial row (tree.py:253)
  }
}

// ------------------------------------------------------------------ K3 accum_probe

__global__ void __launch_bounds__(128) k_accum_probe(vp_tree T, vp_work W, int level, u32 stamp) {
  __shared__ double s_rew[128];
  const int n = W.n;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = r < n;
  if (blockIdx.x == 0 && threadIdx.x == 0) W.level_base[2 * level + 1] = T.counters[0];
  int id = 0;
  double rw = 0.0;
  u32 o = 0;
  if (active) {
    const u32 sl = (u32)W.slot_a[r] & ~kExistBit;
    id = (int)slots(T.hash_a)[sl].id;
    rw = W.reward[r];
    o = W.obs[r];
    if (W.trace_anode) W.trace_anode[(size_t)level * n + r] = id;
  }
  const bool ok = active && id < T.cap_actions;
  // claim (anode, obs) in hash_b first: it is the longest dependent chain
  const u64 key = ((u64)(u32)id << 32) | o;
  const u32 word = warp_claim(slots(T.hash_b), T.hmask_b, key, (u32)r, ok);
  if (active) W.slot_b[r] = (int)word;
  // warp-aggregated reward / visit accumulation, lane (= row) order inside a group
  s_rew[threadIdx.x] = rw;
  __syncwarp();
  const u32 grp = __match_any_sync(FULL, ok ? (u32)id : 0xffffffffu);
  const int leader = __ffs(grp) - 1;
  if (ok && lane_id() == leader) {
    double sum = 0.0;
    u32 g = grp;
    const int wbase = threadIdx.x & ~31;
    while (g) {
      const int l2 = __ffs(g) - 1;
      g &= g - 1;
      sum += s_rew[wbase + l2];
    }
    atomicAdd(&T.a_reward[id], sum);
    atomicAdd(&T.a_visits[id], __popc(grp));
    if (atomicExch(&T.a_stamp[id], stamp) != stamp) {
      const int pos = atomicAdd(&W.pcount[level], 1);
      W.plist[(size_t)level * n + pos] = id;
    }
  }
}

// ------------------------------------------------------------------ leaves

template <class Model>
__global__ void __launch_bounds__(128) k_leaf(vp_tree T, vp_model M, vp_work W, vp_search_args S, int dmax,
                                              u32 stamp) {
  __shared__ double s_h[128];
  const int n = W.n;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = r < n;
  int b = 0;
  double h = 0.0;
  if (active) {
    b = frontier_of(T, W, S, dmax, r);
    h = Model::heuristic(M, reinterpret_cast<const typename Model::State*>(W.states)[r]);
    W.leaf_belief[r] = b;
    W.leaf_value[r] = h;
  }
  const bool ok = active && b < T.cap_beliefs;
  warp_list_once(T.b_stamp, b, stamp, ok, &W.fcount[dmax], W.flist + (size_t)dmax * n);
  s_h[threadIdx.x] = h;
  __syncwarp();
  const u32 grp = __match_any_sync(FULL, ok ? (u32)b : 0xffffffffu);
  const int leader = __ffs(grp) - 1;
  if (ok && lane_id() == leader) {
    double sum = 0.0;
    u32 g = grp;
    const int wbase = threadIdx.x & ~31;
    while (g) {
      const int l2 = __ffs(g) - 1;
      g &= g - 1;
      sum += s_h[wbase + l2];
    }
    atomicAdd(&T.b_weight[b], (double)__popc(grp));
    atomicAdd(&T.b_value[b], sum);
  }
}

// ------------------------------------------------------------------ backup

// Leaves: V = mean heuristic, N = batch count (backup.py:44-51, 82-87), then
// feed the parent action's visit-weighted child mean (backup.py:64-68).
// Warps with spare work materialise the fresh PSI rows of level `mat`
// (the parents the next launch updates).
template <class PsiT>
__global__ void k_backup_leaves(vp_tree T, vp_work W, int dmax, int mat) {
  const int cnt = W.fcount[dmax];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const int b = W.flist[(size_t)dmax * W.n + i];
    const double w = T.b_weight[b];
    const double v = T.b_value[b] / w;
    T.b_value[b] = 0.0;
    T.b_weight[b] = 0.0;
    const int pa = T.b_parent_action[b];
    if (pa >= 0) {
      atomicAdd(&T.a_num[pa], v * w);
      atomicAdd(&T.a_den[pa], w);
    }
  }
  if (mat >= 0) {
    const int mc = W.fcount[mat];
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = gw; i < mc; i += nw) warp_materialise<PsiT>(T, W.flist[(size_t)mat * W.n + i]);
  }
}

template <class PsiT>
__global__ void k_materialise(vp_tree T, vp_work W, int lvl) {
  const int mc = W.fcount[lvl];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < mc; i += nw) warp_materialise<PsiT>(T, W.flist[(size_t)lvl * W.n + i]);
}

// Level d: actions of level d-1 -> Q -> PSI[b, a] += Q - LSE_pre(b)
// (backup.py:96-108); N(b) += lifetime visits (backup.py:110-114).
template <class PsiT>
__global__ void k_backup_q(vp_tree T, vp_work W, int lvl, double gamma) {
  const int cnt = W.pcount[lvl];
  PsiT* psi = reinterpret_cast<PsiT*>(T.psi);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const int a = W.plist[(size_t)lvl * W.n + i];
    const double vis = (double)T.a_visits[a];
    const double q = T.a_reward[a] / vis + (gamma * T.a_num[a]) / T.a_den[a];
    T.a_num[a] = 0.0;
    T.a_den[a] = 0.0;
    const int b = T.a_parent_belief[a];
    PsiT* cell = psi + (size_t)b * T.psi_stride + T.a_action[a];
    *cell = (PsiT)((double)*cell + (q - T.b_lse[b]));
    atomicAdd(&T.b_weight[b], vis);
  }
}

// Level d: beliefs of level d-1 -> V = LSE_post (backup.py:109), cached as
// the next LSE_pre, then their own parent action's child mean (level d-1);
// spare warps materialise the fresh rows of level `mat` = d-2.
template <class PsiT, bool Exact>
__global__ void k_backup_v(vp_tree T, vp_work W, int lvl, int mat) {
  const int cnt = W.fcount[lvl];
  const PsiT* psi = reinterpret_cast<const PsiT*>(T.psi);
  const int A = T.action_count;
  const int lane = lane_id();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  if constexpr (Exact) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
      const int b = W.flist[(size_t)lvl * W.n + i];
      const double v = lse_exact(reinterpret_cast<const double*>(psi) + (size_t)b * T.psi_stride, A, T.eta);
      T.b_lse[b] = v;
      const double w = T.b_weight[b];
      T.b_weight[b] = 0.0;
      const int pa = T.b_parent_action[b];
      if (pa >= 0) {
        atomicAdd(&T.a_num[pa], v * w);
        atomicAdd(&T.a_den[pa], w);
      }
    }
  } else {
    for (int i = gw; i < cnt; i += nw) {
      const int b = W.flist[(size_t)lvl * W.n + i];
      const double v = warp_lse_fast<PsiT>(psi + (size_t)b * T.psi_stride, A, T.eta);
      if (lane == 0) {
        T.b_lse[b] = v;
        const double w = T.b_weight[b];
        T.b_weight[b] = 0.0;
        const int pa = T.b_parent_action[b];
        if (pa >= 0) {
          atomicAdd(&T.a_num[pa], v * w);
          atomicAdd(&T.a_den[pa], w);
        }
      }
    }
  }
  if (mat >= 0) {
    const int mc = W.fcount[mat];
    for (int i = gw; i < mc; i += nw) warp_materialise<PsiT>(T, W.flist[(size_t)mat * W.n + i]);
  }
}

// Levels at or above the search start depth have no recorded lists: derive
// them from the valued children (backup.py:90-95): P_{d-1} = distinct parent
// actions of F_d, F_{d-1} = their distinct parent beliefs.
__global__ void k_parent_lists(vp_tree T, vp_work W, int d, u32 stamp) {
  const int cnt = W.fcount[d];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const int b = W.flist[(size_t)d * W.n + i];
    const int pa = T.b_parent_action[b];
    if (pa < 0) continue;
    if (atomicExch(&T.a_stamp[pa], stamp) != stamp) {
      const int pos = atomicAdd(&W.pcount[d - 1], 1);
      W.plist[(size_t)(d - 1) * W.n + pos] = pa;
      const int pb = T.a_parent_belief[pa];
      if (atomicExch(&T.b_stamp[pb], stamp) != stamp) {
        const int q = atomicAdd(&W.fcount[d - 1], 1);
        W.flist[(size_t)(d - 1) * W.n + q] = pb;
      }
    }
  }
}

template <class PsiT>
__global__ void k_root_argmax(vp_tree T, int* out) {
  const PsiT* row = reinterpret_cast<const PsiT*>(T.psi);
  const int A = T.action_count;
  const int lane = lane_id();
  PsiT best = -(PsiT)INFINITY;
  int arg = A;
  for (int a = lane; a < A; a += 32) {
    const PsiT v = row[a];
    if (v > best) {
      best = v;
      arg = a;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const PsiT vb = __shfl_xor_sync(FULL, best, o);
    const int ab = __shfl_xor_sync(FULL, arg, o);
    if (vb > best || (vb == best && ab < arg)) {
      best = vb;
      arg = ab;
    }
  }
  if (lane == 0) out[0] = arg < A ? arg : 0;
}

__global__ void k_copy_counters(vp_tree T, int* out) {
  if (threadIdx.x < 3) out[1 + threadIdx.x] = T.counters[threadIdx.x];
}

// ------------------------------------------------------------------ test hooks

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
    const double v = warp_lse_fast<PsiT>(rows + (size_t)gw * width, width, eta);
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
    const PsiT e2 = (PsiT)(eta * 1.4426950408889634), sh2 = (PsiT)(eta * lse[g] * 1.4426950408889634);
    out[i] = scan_cdf_scalar<PsiT>(rows + (size_t)g * width, width, e2, sh2, (PsiT)u[i]);
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
  KK_BACKUP_LEAVES, KK_BACKUP_Q, KK_BACKUP_V, KK_PARENT_LISTS, KK_ARGMAX, KK_TREE_INIT, KK_REHASH, KK_COUNT
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

static int stage_budget_bytes() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VP_STAGE_KB");
    v = (e ? atoi(e) : 200) * 1024;
    if (v < 16 * 1024) v = 16 * 1024;
    if (v > 220 * 1024) v = 220 * 1024;
  }
  return v;
}

template <class PsiT>
static StageCfg stage_cfg(int A) {
  int chunks = (int)(((size_t)A * sizeof(PsiT) + 15) / 16);
  if ((chunks & 1) == 0) ++chunks;  // odd number of 16-B chunks: conflict-free LDS.128 across rows
  StageCfg c;
  c.stride = chunks * 16 / (int)sizeof(PsiT);
  const int per_warp = stage_budget_bytes() / 4;
  c.rows = std::max(1, std::min(32, per_warp / (chunks * 16)));
  return c;
}

template <class Model, class PsiT, bool Exact>
static int32_t set_stage_attr(const vp_tree& T) {
  if constexpr (!Exact) {
    const StageCfg sc = stage_cfg<PsiT>(T.action_count);
    const size_t smem = (size_t)4 * sc.rows * sc.stride * sizeof(PsiT);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_level_sample<Model, PsiT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      return VP_ERR_CUDA;
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
  StageCfg sc{0, 0};
  size_t smem = 0;
  if constexpr (!Exact) {
    sc = stage_cfg<PsiT>(T.action_count);
    smem = (size_t)4 * sc.rows * sc.stride * sizeof(PsiT);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusNone) {
      if (int32_t rc = set_stage_attr<Model, PsiT, Exact>(T)) return rc;
    }
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


// Everything one fixed-iteration planning step does on the device, in stream
// order: inputs H2D, fresh tree, per iteration {root draw, search, backup},
// root argmax, counters, result D2H.
template <class Model, class PsiT, bool Exact>
static int32_t enqueue_plan(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_plan_args& P,
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
  { Launch L_(KK_TREE_INIT, st); k_tree_init<PsiT, Exact><<<1, 256, 0, st>>>(T); }
  const u64* keys = reinterpret_cast<const u64*>(P.keys_dev);
  int d = 1;
  for (int it = 0; it < P.iterations; ++it) {
    {
      Launch L_(KK_DRAW, st);
      k_draw<Model><<<blocks_for(W.n, 256), 256, 0, st>>>(W, reinterpret_cast<const State*>(P.particles_dev),
                                                         P.cumw_dev, P.m, 0ull, keys + 2 * it);
    }
    vp_search_args S;
    memset(&S, 0, sizeof(S));
    S.search_key_dev = P.keys_dev + 2 * it + 1;
    S.depth0 = 0;
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

template <class Model, class PsiT, bool Exact>
static int32_t run_plan(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_plan_args& P,
                        cudaStream_t st) {
  int32_t rc = set_stage_attr<Model, PsiT, Exact>(T);
  if (rc) return rc;
  if (!P.use_graph || g_prof_on) return enqueue_plan<Model, PsiT, Exact>(T, M, W, P, st);
  std::vector<unsigned char> key;
  append_pod(key, T);
  append_pod(key, M);
  append_pod(key, W);
  append_pod(key, P);
  const int budget = stage_budget_bytes();
  append_pod(key, budget);
  GraphEntry* hit = nullptr;
  for (auto& e : g_graphs)
    if (e.key == key) hit = &e;
  if (!hit) {
    if (!g_capture_stream && cudaStreamCreateWithFlags(&g_capture_stream, cudaStreamNonBlocking) != cudaSuccess)
      return VP_ERR_CUDA;
    // order the capture stream after the caller's pending work (e.g. init_prefs upload)
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, st);
    cudaStreamWaitEvent(g_capture_stream, ev, 0);
    cudaEventDestroy(ev);
    cudaStreamSynchronize(g_capture_stream);
    const long long l0 = g_launches;
    if (cudaStreamBeginCapture(g_capture_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return VP_ERR_CUDA;
    rc = enqueue_plan<Model, PsiT, Exact>(T, M, W, P, g_capture_stream);
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
    if (g_graphs.size() >= 16) {  // evict the least recently used graph
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
