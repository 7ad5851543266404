// vp_phases.cuh -- the phases of one PORPP planning step as __device__
// functions over a grid-stride index space.  They run either as individual
// kernels (the API path: vp_search / vp_backup, one launch per phase) or back
// to back inside the persistent planning kernel (vp_plan), separated by grid
// barriers.  Every phase is bound by HBM latency / bandwidth; nothing here is
// a dense contraction.
//
// Phase map (reference: /root/reference/pkg/src/vecpomdp):
//   draw        belief.py:37-44        root states for the n rows
//   sample      search.py:107-115      frontier -> softmax draw -> G(s,a) -> claim (b,a)
//   assign<0>   tree.py:180-218        number new action rows in first-occurrence order
//   accum       tree.py:216-217,236    reward/visit sums, claim (anode, obs)
//   assign<1>   tree.py:220-256        number new belief rows in first-occurrence order
//   leaf        search.py:119, backup.py:44-51
//   backup_*    backup.py:75-114       leaf means, Q + PSI scatter, LSE per level
#pragma once

#include <type_traits>

#include "vp_common.cuh"
#include "vp_models.cuh"

namespace vp {

constexpr int kStageWarps = 8;  // warps per block of the persistent kernel

__device__ __forceinline__ Slot* slots(void* p) { return reinterpret_cast<Slot*>(p); }

// Grid-stride execution context.
struct Span {
  int gtid, gthreads;  // thread index / count
  int gwarp, gwarps;   // warp index / count
};
// Warps are numbered block-fastest (warp w of block b is global warp
// w * gridDim + b) so that consecutive 32-row chunks land on different SMs
// even when a phase has far fewer chunks than the grid has warps; lanes stay
// contiguous, so thread-granular loops remain coalesced.
__device__ __forceinline__ Span this_span() {
  Span s;
  s.gwarp = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  s.gwarps = (blockDim.x >> 5) * gridDim.x;
  s.gtid = s.gwarp * 32 + (threadIdx.x & 31);
  s.gthreads = s.gwarps * 32;
  return s;
}

// ------------------------------------------------------------------ exp helpers (fast mode)
// exp(eta * psi - shift) is evaluated as exp2(fma(eta*log2e, psi, -shift*log2e)).
__device__ __forceinline__ float fexp2(float x) { return exp2f(x); }
__device__ __forceinline__ double fexp2(double x) { return exp2(x); }
__device__ __forceinline__ float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double ffma(double a, double b, double c) { return __fma_rn(a, b, c); }
constexpr double kLog2eD = 1.4426950408889634;

// ------------------------------------------------------------------ LSE

// Fast LSE (backup.py:34-41 formula: max, then sum of exp), evaluated by a
// group of lanes per row with the row held in registers.
__device__ __forceinline__ double lse_log(float s) { return (double)logf(s); }
__device__ __forceinline__ double lse_log(double s) { return log(s); }

// Sub-warp LSE: a group of G lanes (G a power of two) per row, so short rows
// (|A| <= 16 G) keep every lane busy and take one memory round trip.  All
// 32 lanes must call it (rows may be null for idle groups).
__host__ __device__ constexpr int lse_group_size(int A) {
  return A <= 16 ? 1 : A <= 32 ? 2 : A <= 64 ? 4 : A <= 128 ? 8 : A <= 256 ? 16 : 32;
}

template <class PsiT, int G>
__device__ __forceinline__ double lse_group(const PsiT* row, int A, double eta) {
  const int gl = lane_id() & (G - 1);
  constexpr int R = 16;
  const PsiT e = (PsiT)eta;
  const PsiT e2 = (PsiT)(eta * kLog2eD);
  PsiT m = -(PsiT)INFINITY, s = 0;
  if (A <= G * R) {
    PsiT v[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int a = gl + G * k;
      v[k] = (row && a < A) ? row[a] : -(PsiT)INFINITY;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const PsiT z = e * v[k];
      m = z > m ? z : m;
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const PsiT w = __shfl_xor_sync(FULL, m, o, G);
      m = w > m ? w : m;
    }
    const PsiT m2 = m * (PsiT)kLog2eD;
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (row && gl + G * k < A) s += fexp2(ffma(e2, v[k], -m2));
  } else {
    if (row)
      for (int a = gl; a < A; a += G) {
        const PsiT z = e * row[a];
        m = z > m ? z : m;
      }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const PsiT w = __shfl_xor_sync(FULL, m, o, G);
      m = w > m ? w : m;
    }
    const PsiT m2 = m * (PsiT)kLog2eD;
    if (row)
      for (int a = gl; a < A; a += G) s += fexp2(ffma(e2, row[a], -m2));
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o, G);
  return (double)m / eta + lse_log(s) / eta;
}

// Runtime dispatch of the group size; f is called as f(std::integral_constant<int, G>()).
template <class F>
__device__ __forceinline__ void with_group(int A, const F& f) {
  switch (lse_group_size(A)) {
    case 1: f(std::integral_constant<int, 1>()); break;
    case 2: f(std::integral_constant<int, 2>()); break;
    case 4: f(std::integral_constant<int, 4>()); break;
    case 8: f(std::integral_constant<int, 8>()); break;
    case 16: f(std::integral_constant<int, 16>()); break;
    default: f(std::integral_constant<int, 32>()); break;
  }
}

// The fast LSE of one row as the tree caches it (group size from |A|); called by a full warp.
template <class PsiT>
__device__ double row_lse_fast(const PsiT* row, int A, double eta) {
  double out = 0.0;
  with_group(A, [&](auto g) {
    constexpr int G = decltype(g)::value;
    const double v = lse_group<PsiT, G>(lane_id() < G ? row : nullptr, A, eta);
    out = __shfl_sync(FULL, v, 0);
  });
  return out;
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

// Fast draw: probabilities exp(eta (psi - LSE)) with the row's cached LSE,
// accumulated left to right until the running sum exceeds u (clamp |A|-1,
// search.py:83).  Scalar and vectorised versions do the same fp sequence.
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

struct StageCfg {
  int rows;    // G: PSI rows staged per warp per batch
  int stride;  // staged row stride in PsiT elements (odd multiple of 16 bytes)
};

// Per-warp staging state carried across phases of the persistent kernel.
template <class PsiT>
struct Stage {
  PsiT* buf;
  u64* bar;
  u32 phase;
  StageCfg cfg;
};

// ------------------------------------------------------------------ warp helpers

// Lanes with equal keys elect their lowest lane (= smallest row) to probe or
// claim the slot once; the slot word is broadcast back.
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

// Append `node` to a per-level list once per level (stamp dedup).  Returns
// true on the lane that appended it.
__device__ __forceinline__ bool warp_list_once(u32* stamp, int node, u32 value, bool active, int* count, int* list) {
  const u32 grp = __match_any_sync(FULL, active ? (u32)node : 0xffffffffu);
  const int leader = __ffs(grp) - 1;
  bool added = false;
  if (active && lane_id() == leader) {
    if (atomicExch(&stamp[node], value) != value) {
      const int pos = atomicAdd(count, 1);
      list[pos] = node;
      added = true;
    }
  }
  return added;
}

// Id of a slot once its first-occurrence row has numbered it (spin while pending).
// Relaxed spin: the id's publisher stores it with st.release after the node's
// columns, and readers only touch those columns through addresses that
// depend on the id (or with relaxed gpu-scope loads).
__device__ __forceinline__ int wait_final(const Slot* tab, u32 slot_word) {
  const u32* p = &tab[slot_word & ~kExistBit].id;
  u32 v = ld_relaxed_u32(p);
  while (v >= kPending) v = ld_relaxed_u32(p);
  return (int)v;
}

// Sum of v over the lanes in `grp`, in lane (= row) order, delivered to all lanes.
__device__ __forceinline__ double group_sum_ordered(double v, u32 grp) {
  double s = 0.0;
#pragma unroll 4
  for (int j = 0; j < 32; ++j) {
    const double x = __shfl_sync(FULL, v, j);
    if ((grp >> j) & 1u) s += x;
  }
  return s;
}

// Write the initial PSI row into every still-fresh belief of list[0..cnt)
// (lazy rows, tree.py:253); a group of G lanes per belief.
template <class PsiT>
__device__ void materialise_list(const vp_tree& T, const int* list, int cnt, const Span& sp) {
  const int A = T.action_count;
  with_group(A, [&](auto g) {
    constexpr int G = decltype(g)::value;
    constexpr int RPW = 32 / G;
    const int gl = lane_id() & (G - 1), grp = lane_id() / G;
    for (int i0 = sp.gwarp * RPW; i0 < cnt; i0 += sp.gwarps * RPW) {
      const int i = i0 + grp;
      if (i >= cnt) continue;
      const int b = list[i];
      if (!(T.b_flags[b] & 1)) continue;
      PsiT* row = reinterpret_cast<PsiT*>(T.psi) + (size_t)b * T.psi_stride;
      for (int a = gl; a < A; a += G) row[a] = (PsiT)T.init_prefs[a];
      if (gl == 0) T.b_flags[b] = 0;
    }
  });
}

// ------------------------------------------------------------------ tree init (one block)

template <class PsiT, bool Exact>
__device__ void block_tree_init(const vp_tree& T) {
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
      v = row_lse_fast<PsiT>(psi, A, T.eta);
    }
    if (threadIdx.x == 0) {
      T.init_lse[0] = v;
      T.b_lse[0] = v;
      // CDF of the initial row with the fast sampler's exact arithmetic
      PsiT* cdf = reinterpret_cast<PsiT*>(T.init_cdf);
      const PsiT e2 = (PsiT)(T.eta * kLog2eD), sh2 = (PsiT)(T.eta * v * kLog2eD);
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
  __syncthreads();
}

// ------------------------------------------------------------------ draw

template <class Model>
__device__ void phase_draw(const vp_work& W, const typename Model::State* particles, const double* cumw, int m,
                           u64 key, const Span& sp) {
  for (int r = sp.gtid; r < W.n; r += sp.gthreads) {
    const double u = uniform1(key, (u64)r);
    int lo = 0, hi = m;  // first index with cum > u  (searchsorted side=right)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cumw[mid] > u) hi = mid;
      else lo = mid + 1;
    }
    const int idx = lo < m - 1 ? lo : m - 1;
    reinterpret_cast<typename Model::State*>(W.states)[r] = particles[idx];
  }
}

// ------------------------------------------------------------------ sample (K1)

struct LevelArgs {
  int level;
  int depth0;
  u64 lkey;       // search_rng.derive(level).key (search.py:107)
  u32 stamp;
  const int32_t* inject;  // [*, n] level-major, or null
  const int32_t* start;   // [n] frontier at depth0, or null (root)
};

__device__ __forceinline__ int frontier_of(const vp_tree& T, const vp_work& W, const LevelArgs& L, int r) {
  if (L.level == L.depth0) return L.start ? L.start[r] : 0;
  const int b = wait_final(slots(T.hash_b), (u32)W.slot_b[r]);
  if (W.trace_belief) W.trace_belief[(size_t)(L.level - 1) * W.n + r] = b;
  return b;
}

template <class Model>
__device__ __forceinline__ void step_and_claim(const vp_tree& T, const vp_model& M, const vp_work& W,
                                               const LevelArgs& L, int r, bool active, int b, int a) {
  u64 key = 0;
  if (active) {
    typename Model::State st = reinterpret_cast<typename Model::State*>(W.states)[r];
    u32 o;
    double rw;
    Model::step(M, st, a, fold(L.lkey, 1), (u64)r, o, rw);  // level_rng.derive(1) (search.py:113-115)
    reinterpret_cast<typename Model::State*>(W.states)[r] = st;
    W.obs[r] = o;
    W.reward[r] = rw;
    W.action[r] = a;
    if (W.trace_action) {
      W.trace_action[(size_t)L.level * W.n + r] = a;
      W.trace_obs[(size_t)L.level * W.n + r] = o;
    }
    key = ((u64)(u32)b << 32) | (u32)a;
  }
  const u32 word = warp_claim(slots(T.hash_a), T.hmask_a, key, (u32)r, active);
  if (active) W.slot_a[r] = (int)word;
}

// Fast mode: warps take 32-row chunks.  Rows whose belief is fresh draw from
// the shared initial CDF; the chunk's distinct non-fresh beliefs have their
// PSI rows TMA bulk-copied into the warp's shared-memory stage (one
// cp.async.bulk per row, completion on the warp's mbarrier) and every lane
// scans its own row.
template <class Model, class PsiT>
__device__ void phase_sample_fast(const vp_tree& T, const vp_model& M, const vp_work& W, const LevelArgs& L,
                                  Stage<PsiT>& sg, PsiT* init_cdf, const Span& sp) {
  const int n = W.n, A = T.action_count, lane = lane_id();
  if (W.stats && sp.gtid == 0) {
    atomicAdd(&W.stats[3], 1ull);
    atomicAdd(&W.stats[4], (unsigned long long)n);
  }
  // the shared initial-row CDF (fresh beliefs) lives in shared memory
  for (int a = threadIdx.x; a < A; a += blockDim.x) init_cdf[a] = reinterpret_cast<const PsiT*>(T.init_cdf)[a];
  __syncthreads();
  if (sp.gtid == 0) W.level_base[2 * L.level] = T.counters[1];
  const PsiT* psi = reinterpret_cast<const PsiT*>(T.psi);
  const u32 row_bytes = (u32)(((size_t)A * sizeof(PsiT) + 15) & ~(size_t)15);
  const PsiT e2 = (PsiT)(T.eta * kLog2eD);
  for (int c = sp.gwarp; c * 32 < n; c += sp.gwarps) {
    const int r = c * 32 + lane;
    const bool active = r < n;
    const int b = active ? frontier_of(T, W, L, r) : 0;
    warp_list_once(T.b_stamp, b, L.stamp, active, &W.fcount[L.level], W.flist + (size_t)L.level * n);
    const double u = active ? uniform1(fold(L.lkey, 0), (u64)r) : 0.0;  // level_rng.derive(0) (search.py:110)
    int a = 0;
    if (L.inject) {
      a = active ? L.inject[(size_t)L.level * n + r] : 0;
    } else {
      const bool fresh = active && (ld_relaxed_u8(&T.b_flags[b]) & 1);
      const bool need = active && !fresh;
      if (fresh) a = search_cdf(init_cdf, A, (PsiT)u);
      const u32 grp = __match_any_sync(FULL, need ? (u32)b : 0xffffffffu);
      const int my_leader = __ffs(grp) - 1;
      const u32 leaders = __ballot_sync(FULL, need && lane == my_leader);
      const int K = __popc(leaders);
      if (W.stats && lane == 0 && K) atomicAdd(&W.stats[2], (unsigned long long)K);
      const int my_slot = need ? __popc(leaders & ((1u << my_leader) - 1u)) : -1;
      const PsiT sh2 = need ? (PsiT)(T.eta * ld_relaxed_f64(&T.b_lse[b]) * kLog2eD) : (PsiT)0;
      for (int s0 = 0; s0 < K; s0 += sg.cfg.rows) {
        const int cnt = min(sg.cfg.rows, K - s0);
        fence_async_smem();
        if (lane == 0) mbar_expect_tx(sg.bar, row_bytes * (u32)cnt);
        __syncwarp();
        const bool mine = need && my_slot >= s0 && my_slot < s0 + cnt;
        if (mine && lane == my_leader)
          bulk_g2s(sg.buf + (size_t)(my_slot - s0) * sg.cfg.stride, psi + (size_t)b * T.psi_stride, row_bytes,
                   sg.bar);
        mbar_wait(sg.bar, sg.phase);
        sg.phase ^= 1u;
        if (mine) a = scan_cdf_vec<PsiT>(sg.buf + (size_t)(my_slot - s0) * sg.cfg.stride, A, e2, sh2, (PsiT)u);
        __syncwarp();
      }
    }
    step_and_claim<Model>(T, M, W, L, r, active, b, a);
  }
}

// fp64 parity mode: numpy operation order, no staging.
template <class Model>
__device__ void phase_sample_exact(const vp_tree& T, const vp_model& M, const vp_work& W, const LevelArgs& L,
                                   const Span& sp) {
  const int n = W.n, A = T.action_count, lane = lane_id();
  if (sp.gtid == 0) W.level_base[2 * L.level] = T.counters[1];
  for (int c = sp.gwarp; c * 32 < n; c += sp.gwarps) {
    const int r = c * 32 + lane;
    const bool active = r < n;
    const int b = active ? frontier_of(T, W, L, r) : 0;
    warp_list_once(T.b_stamp, b, L.stamp, active, &W.fcount[L.level], W.flist + (size_t)L.level * n);
    int a = 0;
    if (active) {
      const double u = uniform1(fold(L.lkey, 0), (u64)r);
      if (L.inject) {
        a = L.inject[(size_t)L.level * n + r];
      } else {
        const double* row = (ld_relaxed_u8(&T.b_flags[b]) & 1)
                                ? T.init_prefs
                                : reinterpret_cast<const double*>(T.psi) + (size_t)b * T.psi_stride;
        a = sample_exact(row, A, T.eta, u);
      }
    }
    step_and_claim<Model>(T, M, W, L, r, active, b, a);
  }
}

// ------------------------------------------------------------------ assign (K2 / K4)

// Number the rows that won their key this level in row order: tiles of
// blockDim.x rows (one per thread), chained by a warp-parallel decoupled
// look-back; write the new nodes' columns and publish the id (release) so
// rows spinning in the next phase can proceed.  Block-collective.
// WhichTable: 0 = actions, 1 = beliefs.
// `ticket` != null (one tile per block, standalone launch): tiles are taken in
// block start order from an atomic ticket, which makes the look-back
// deadlock-free for any grid size; null (persistent kernel, all blocks
// resident): block b owns tiles b, b + grid, ...
template <int WhichTable>
__device__ void phase_assign(const vp_tree& T, const vp_work& W, int level, u32 epoch, u32* ticket) {
  __shared__ u32 s_warp[32];
  __shared__ u32 s_excl;
  __shared__ int s_tile;
  const int n = W.n;
  const int NW = blockDim.x >> 5;
  const int tile_rows = blockDim.x;
  const int ntiles = (n + tile_rows - 1) / tile_rows;
  Slot* tab = slots(WhichTable ? T.hash_b : T.hash_a);
  const int* slot_of = WhichTable ? W.slot_b : W.slot_a;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int base = W.level_base[2 * level + WhichTable];
  const int cap = WhichTable ? T.cap_beliefs : T.cap_actions;
  int first = blockIdx.x;
  if (ticket) {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    first = s_tile;
  }
  const int step = ticket ? ntiles : gridDim.x;
  for (int tile = first; tile < ntiles; tile += step) {
    const int r = tile * tile_rows + threadIdx.x;
    u32 sl = 0;
    bool win = false;
    if (r < n) {
      const u32 w = (u32)slot_of[r];
      sl = w & ~kExistBit;
      if (!(w & kExistBit)) win = ld_volatile_u32(&tab[sl].id) == (kPending | (u32)r);
    }
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
        if (tile == ntiles - 1) {
          if (W.stats) {
            // lists of this level are complete by now: F_l after sample, P_l after accum
            atomicAdd(&W.stats[WhichTable ? 1 : 0],
                      (unsigned long long)(WhichTable ? W.pcount[level] : W.fcount[level]));
            atomicAdd(&W.stats[WhichTable ? 6 : 5], (unsigned long long)(excl + agg));
          }
          T.counters[WhichTable ? 0 : 1] = base + (int)(excl + agg);
          if (ticket) *ticket = 0;  // every block has taken its ticket by now
        }
      }
    }
    __syncthreads();
    if (win) {
      const int id = base + (int)(s_excl + s_warp[warp] + below);
      Slot& s = tab[sl];
      if (id < cap) {
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
      } else {
        T.counters[2] = 1;  // overflow: the host fails the plan loudly
      }
      st_release_u32(&s.id, (u32)id);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ accum (K3)

__device__ void phase_accum(const vp_tree& T, const vp_work& W, int level, u32 stamp, const Span& sp) {
  const int n = W.n, lane = lane_id();
  if (sp.gtid == 0) W.level_base[2 * level + 1] = T.counters[0];
  for (int c = sp.gwarp; c * 32 < n; c += sp.gwarps) {
    const int r = c * 32 + lane;
    const bool active = r < n;
    int id = 0;
    double rw = 0.0;
    u32 o = 0;
    if (active) {
      id = wait_final(slots(T.hash_a), (u32)W.slot_a[r]);
      rw = W.reward[r];
      o = W.obs[r];
      if (W.trace_anode) W.trace_anode[(size_t)level * n + r] = id;
    }
    const bool ok = active && id < T.cap_actions;
    // claim (anode, obs) in hash_b first: it is the longest dependent chain
    const u32 word = warp_claim(slots(T.hash_b), T.hmask_b, ((u64)(u32)id << 32) | o, (u32)r, ok);
    if (active) W.slot_b[r] = (int)word;
    // warp-aggregated reward / visit accumulation (lane = row order inside a group)
    const u32 grp = __match_any_sync(FULL, ok ? (u32)id : 0xffffffffu);
    const double sum = group_sum_ordered(rw, grp);
    if (ok && lane == __ffs(grp) - 1) {
      atomicAdd(&T.a_reward[id], sum);
      atomicAdd(&T.a_visits[id], __popc(grp));
      if (atomicExch(&T.a_stamp[id], stamp) != stamp) {
        const int pos = atomicAdd(&W.pcount[level], 1);
        W.plist[(size_t)level * n + pos] = id;
      }
    }
  }
}

// ------------------------------------------------------------------ leaves

template <class Model>
__device__ void phase_leaf(const vp_tree& T, const vp_model& M, const vp_work& W, const LevelArgs& L,
                           const Span& sp) {
  const int n = W.n, lane = lane_id();
  for (int c = sp.gwarp; c * 32 < n; c += sp.gwarps) {
    const int r = c * 32 + lane;
    const bool active = r < n;
    int b = 0;
    double h = 0.0;
    if (active) {
      b = frontier_of(T, W, L, r);
      h = Model::heuristic(M, reinterpret_cast<const typename Model::State*>(W.states)[r]);
      W.leaf_belief[r] = b;
      W.leaf_value[r] = h;
    }
    const bool ok = active && b < T.cap_beliefs;
    warp_list_once(T.b_stamp, b, L.stamp, ok, &W.fcount[L.level], W.flist + (size_t)L.level * n);
    const u32 grp = __match_any_sync(FULL, ok ? (u32)b : 0xffffffffu);
    const double sum = group_sum_ordered(h, grp);
    if (ok && lane == __ffs(grp) - 1) {
      atomicAdd(&T.b_weight[b], (double)__popc(grp));
      atomicAdd(&T.b_value[b], sum);
    }
  }
}

// ------------------------------------------------------------------ backup

// Leaves: V = mean heuristic, N = batch count (backup.py:44-51, 82-87), fed
// to the parent action's child mean (backup.py:64-68); warps also
// materialise the fresh PSI rows of level `mat` (the parents updated next).
template <class PsiT>
__device__ void phase_backup_leaves(const vp_tree& T, const vp_work& W, int dmax, int mat, const Span& sp) {
  const int cnt = W.fcount[dmax];
  for (int i = sp.gtid; i < cnt; i += sp.gthreads) {
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
  if (mat >= 0) materialise_list<PsiT>(T, W.flist + (size_t)mat * W.n, W.fcount[mat], sp);
}

template <class PsiT>
__device__ void phase_materialise(const vp_tree& T, const vp_work& W, int lvl, const Span& sp) {
  materialise_list<PsiT>(T, W.flist + (size_t)lvl * W.n, W.fcount[lvl], sp);
}

// Actions of level lvl: Q = R/visits + gamma num/den; PSI[b, a] += Q - LSE_pre(b)
// (backup.py:96-108); N(b) += lifetime visits (backup.py:110-114).
template <class PsiT>
__device__ void phase_backup_q(const vp_tree& T, const vp_work& W, int lvl, double gamma, const Span& sp) {
  const int cnt = W.pcount[lvl];
  PsiT* psi = reinterpret_cast<PsiT*>(T.psi);
  for (int i = sp.gtid; i < cnt; i += sp.gthreads) {
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

// Beliefs of level lvl: V = LSE_post (backup.py:109), cached as the next
// LSE_pre, then their parent action's child mean; warps also materialise
// the fresh rows of level `mat`.
template <class PsiT, bool Exact>
__device__ void phase_backup_v(const vp_tree& T, const vp_work& W, int lvl, int mat, const Span& sp) {
  const int cnt = W.fcount[lvl];
  const PsiT* psi = reinterpret_cast<const PsiT*>(T.psi);
  const int A = T.action_count;
  auto finish = [&](int b, double v) {
    T.b_lse[b] = v;
    const double w = T.b_weight[b];
    T.b_weight[b] = 0.0;
    const int pa = T.b_parent_action[b];
    if (pa >= 0) {
      atomicAdd(&T.a_num[pa], v * w);
      atomicAdd(&T.a_den[pa], w);
    }
  };
  if constexpr (Exact) {
    for (int i = sp.gtid; i < cnt; i += sp.gthreads) {
      const int b = W.flist[(size_t)lvl * W.n + i];
      finish(b, lse_exact(reinterpret_cast<const double*>(psi) + (size_t)b * T.psi_stride, A, T.eta));
    }
  } else {
    with_group(A, [&](auto g) {
      constexpr int G = decltype(g)::value;
      constexpr int RPW = 32 / G;  // rows per warp
      const int gl = lane_id() & (G - 1), grp = lane_id() / G;
      for (int i0 = sp.gwarp * RPW; i0 < cnt; i0 += sp.gwarps * RPW) {
        const int i = i0 + grp;
        const int b = i < cnt ? W.flist[(size_t)lvl * W.n + i] : -1;
        const double v = lse_group<PsiT, G>(b >= 0 ? psi + (size_t)b * T.psi_stride : nullptr, A, T.eta);
        if (gl == 0 && b >= 0) finish(b, v);
      }
    });
  }
  if (mat >= 0) materialise_list<PsiT>(T, W.flist + (size_t)mat * W.n, W.fcount[mat], sp);
}

// Levels at or above the search start depth have no recorded lists: derive
// them from the valued children (backup.py:90-95).
__device__ void phase_parent_lists(const vp_tree& T, const vp_work& W, int d, u32 stamp, const Span& sp) {
  const int cnt = W.fcount[d];
  for (int i = sp.gtid; i < cnt; i += sp.gthreads) {
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
__device__ void warp_root_argmax(const vp_tree& T, int* out) {
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

}  // namespace vp
