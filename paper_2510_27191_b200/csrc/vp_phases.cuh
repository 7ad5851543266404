// vp_phases.cuh -- device code of one PORPP planning pass (sm_100a).
//
// A pass is three kernels and no grid barrier:
//
//   search  (search.py:86-119)  each warp carries its 32 rows through every
//           level: softmax draw (the shared initial CDF, an overlay record's
//           corrected CDF, or a dense row's CDF row TMA-staged into shared
//           memory), G(s,a) in registers, the (b,a) and (b,a,o) hash claims --
//           one 128-bit CAS each, issued together, inserting the creator's
//           static id -- and reward / visit / row-count reductions; then the
//           leaf heuristic.  A row never waits for rows of other warps.
//   backup  (backup.py:75-114)  a bottom-up completion wave: every distinct
//           leaf delivers (V, N) to its parent action; the delivery that
//           brings an action's delivered-row count to its row count completes
//           the action (Q, PSI update), and the action completion that does
//           the same for its belief completes the belief (LSE_post without
//           reading the row, save ill-conditioned dense rows) and climbs on.
//   cdf rows  the dense rows the backup changed get their softmax CDF rows.
//
// Node ids are static: row r creating at level l takes id extent + l n + r.
// Each node stores the key (pass, level, first row) under which the reference
// would have created it; the host sorts by it when exporting, which
// reproduces the reference's first-occurrence numbering (tree.py:10-12).
#pragma once

#include <type_traits>

#include "vp_common.cuh"
#include "vp_models.cuh"

namespace vp {

constexpr int kSearchWarps = 4;   // warps per search block (4: C3 -1.5 %, C2 / C5 even against 1 or 2)

// Measurement builds only (-DVP_PHASE_CLOCKS, scripts/phase_clocks.sh): SM cycles per search
// phase summed over warps (lane 0), read back with vp_debug_phases.
#ifdef VP_PHASE_CLOCKS
__device__ unsigned long long g_phase_cycles[24];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// completion trace: (globaltimer mod 2^48) << 16 | pass << 8 | depth, buffered per warp in shared
// memory and flushed once per warp (no contended atomics on the climb)
__device__ unsigned long long g_trace[1 << 21];
__device__ unsigned int g_trace_n;
#define VP_WAVE_DECL() __shared__ unsigned long long s_tr[8][256]; __shared__ int s_trn[8]; \
  const int w_tr = threadIdx.x >> 5; if (lane_id() == 0) s_trn[w_tr] = 0; __syncwarp();
#define VP_WAVE(pass, depth) { const int k_ = atomicAdd(&s_trn[w_tr], 1); \
  if (k_ < 256) s_tr[w_tr][k_] = ((gtimer() & ((1ull << 40) - 1)) << 24) | (((pass) & 63u) << 18) | \
      ((unsigned)(depth) << 12) | ((blockIdx.x * 8 + w_tr) & 4095u); }
#define VP_WAVE_FLUSH() { __syncwarp(); const int n_ = min(s_trn[w_tr], 256); unsigned b_ = 0; \
  if (lane_id() == 0) b_ = atomicAdd(&g_trace_n, (unsigned)n_); b_ = __shfl_sync(FULL, b_, 0); \
  for (int i_ = lane_id(); i_ < n_; i_ += 32) if (b_ + i_ < (1u << 21)) g_trace[b_ + i_] = s_tr[w_tr][i_]; }
#define VP_PH_INIT() long long ph_t0 = clock64(); unsigned long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define VP_PH(k) { const long long t_ = clock64(); ph_acc[k] += (unsigned long long)(t_ - ph_t0); ph_t0 = t_; }
#define VP_PH_FLUSH() if (lane_id() == 0) for (int k_ = 0; k_ < 8; ++k_) atomicAdd(&g_phase_cycles[k_], ph_acc[k_]);
#define VP_BK(k) { const long long t_ = clock64(); if (lane_id() == 0) atomicAdd(&g_phase_cycles[16 + k], (unsigned long long)(t_ - bk_t0)); bk_t0 = clock64(); }
#define VP_BK_INIT() long long bk_t0 = clock64();
#define VP_DR_INIT() long long dr_t0 = clock64();
#define VP_DR(k) { const long long t_ = clock64(); if (lane_id() == 0) atomicAdd(&g_phase_cycles[8 + k], (unsigned long long)(t_ - dr_t0)); dr_t0 = clock64(); }
#else
#define VP_DR_INIT()
#define VP_DR(k)
#define VP_WAVE(pass, depth)
#define VP_WAVE_DECL()
#define VP_WAVE_FLUSH()
#define VP_BK_INIT()
#define VP_BK(k)
#define VP_PH_INIT()
#define VP_PH(k)
#define VP_PH_FLUSH()
#endif
constexpr int kBackupWarps = 8;   // warps per backup block

__device__ __forceinline__ Slot* slots(void* p) { return reinterpret_cast<Slot*>(p); }

// Canonical creation key: the reference creates node ids pass by pass, level
// by level, in first-occurrence row order (tree.py:180-256).
__device__ __forceinline__ u64 creation_key(u32 pass, int level, int row) {
  return ((u64)pass << 32) | ((u64)(u32)level << 24) | (u64)(u32)row;
}

// Key of belief node (parent belief b, action a -> action row x, observation o)
// in the belief index: mode 1 does not need x, so a level can issue its action
// and belief claims together (vp_tree.bkey_mode).
__device__ __forceinline__ u64 belief_key(const vp_tree& T, int b, int a, int x, u32 o) {
  return T.bkey_mode ? (((u64)(u32)b << 32) | ((u64)(u32)a << 20) | (u64)o) : (((u64)(u32)x << 32) | (u64)o);
}

// Two-phase claim: the first CAS of a probe sequence (predicated, no branch, so a
// warp can have several claims in flight), then the rest of the probe loop.
struct ClaimTry {
  u64 h, old_key, old_word;
};
__device__ __forceinline__ ClaimTry claim_try(Slot* tab, u64 mask, u64 key, bool go) {
  ClaimTry t{slot_hash(key) & mask, kEmptyKey, ~0ull};
  if (go) cas128(&tab[t.h], kEmptyKey, ~0ull, key, ~0ull, t.old_key, t.old_word);
  return t;
}
// Claims that insert the creator's id with the key ({key, pass << 32 | id} in the CAS): the id
// is known before the claim (static per-row numbering), so a slot is never unpublished and a
// hit returns the node in the same round trip.
__device__ __forceinline__ ClaimTry claim_try_id(Slot* tab, u64 mask, u64 key, u64 word, bool go) {
  ClaimTry t{slot_hash(key) & mask, kEmptyKey, ~0ull};
  if (go) cas128(&tab[t.h], kEmptyKey, ~0ull, key, word, t.old_key, t.old_word);
  return t;
}
__device__ __forceinline__ Claim claim_finish_id(Slot* tab, u64 mask, u64 key, u64 word, ClaimTry t) {
  u64 h = t.h, old_key = t.old_key, old_word = t.old_word;
  while (true) {
    if (old_key == kEmptyKey) return Claim{(u32)h, true, word};
    if (old_key == key) return Claim{(u32)h, false, old_word};
    h = (h + 1) & mask;
    cas128(&tab[h], kEmptyKey, ~0ull, key, word, old_key, old_word);
  }
}
__device__ __forceinline__ Claim claim_finish(Slot* tab, u64 mask, u64 key, ClaimTry t) {
  u64 h = t.h, old_key = t.old_key, old_word = t.old_word;
  while (true) {
    if (old_key == kEmptyKey) return Claim{(u32)h, true, ~0ull};
    if (old_key == key) return Claim{(u32)h, false, old_word};
    h = (h + 1) & mask;
    cas128(&tab[h], kEmptyKey, ~0ull, key, ~0ull, old_key, old_word);
  }
}

// Backup accumulator of a node: sum (V*N for an action, the incremental
// exp-sum for a belief), rows delivered so far, and an integer count (sum N
// for an action, lifetime visits of the valued actions for a belief).
struct __align__(16) Acc {
  double sum;
  u32 rows;
  u32 cnt;
};

// Deliver (dsum, drows, dcnt) to a node whose deliveries total `target` rows.
// Returns true on the completing delivery, with the totals in `out`.
//  * A delivery carrying all of the node's rows is its only one: no atomic.
//  * A node with few rows (target <= kCasRows) sees few, rarely concurrent
//    deliveries: ONE optimistic 128-bit CAS on {sum, rows, cnt} (guess: still
//    zero), retried from the returned value; the completing CAS returns the
//    totals -- no fence, no reload.
//  * Busy nodes (the top of the tree) take many concurrent deliveries: L2
//    reductions of the sums, then an acq_rel add on the row count elects the
//    completing delivery, which reads the totals.
// The path depends only on `target`, so all deliveries to a node agree on it.
constexpr u32 kCasRows = 16;
// Row counts are < 2^24 (n_parallel < 2^24): the top 8 bits of a delivery's row count are
// free for flags that add up like a bit-or (each set by exactly one delivery of the pass) --
// the overlay slots an action completion changed (kSlotBit << slot).
constexpr u32 kRowsMask = 0xFFFFFFu;
constexpr u32 kSlotBit = 1u << 24;

__device__ __forceinline__ void cas128_acq_rel(void* p, u64 cmp_lo, u64 cmp_hi, u64 new_lo, u64 new_hi, u64& old_lo,
                                               u64& old_hi) {
  asm volatile(
      "{\n .reg .b128 c, n, d;\n mov.b128 c, {%2, %3};\n mov.b128 n, {%4, %5};\n"
      " atom.acq_rel.gpu.global.cas.b128 d, [%6], c, n;\n mov.b128 {%0, %1}, d;\n}\n"
      : "=l"(old_lo), "=l"(old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(new_lo), "l"(new_hi), "l"(p)
      : "memory");
}

// `ordered`: the deliveries also publish the deliverer's earlier stores to the completing one
// (a dense PSI cell its full-row fallback may read): the CAS path then runs acq_rel; the busy
// path's row-count add is acq_rel anyway, and a lone delivery is its own completer.
template <bool ordered = false>
__device__ __forceinline__ bool acc_deliver(void* base, int i, double dsum, u32 drows, u32 dcnt, u32 target,
                                            Acc& out) {
  if ((drows & kRowsMask) == target) {
    out = Acc{dsum, drows, dcnt};
    return true;
  }
  Acc* p = reinterpret_cast<Acc*>(base) + i;
  if (target <= kCasRows) {
    u64 lo = 0, hi = 0;
    while (true) {
      const double s = __longlong_as_double((long long)lo) + dsum;
      const u32 r = (u32)hi + drows, c = (u32)(hi >> 32) + dcnt;
      const u64 nlo = (u64)__double_as_longlong(s), nhi = (u64)r | ((u64)c << 32);
      u64 olo, ohi;
      if (ordered) cas128_acq_rel(p, lo, hi, nlo, nhi, olo, ohi);
      else cas128(p, lo, hi, nlo, nhi, olo, ohi);
      if (olo == lo && ohi == hi) {
        if ((r & kRowsMask) != target) return false;
        out = Acc{s, r, c};
        *p = Acc{0.0, 0u, 0u};
        return true;
      }
      lo = olo;
      hi = ohi;
    }
  }
  red_add(&p->sum, dsum);
  red_add(reinterpret_cast<int*>(&p->cnt), (int)dcnt);
  const u32 rows = (u32)atom_add_acq_rel(reinterpret_cast<int*>(&p->rows), (int)drows) + drows;
  if ((rows & kRowsMask) != target) return false;
  out.sum = ld_relaxed_f64(&p->sum);
  out.cnt = ld_relaxed_u32(&p->cnt);
  out.rows = rows;
  *p = Acc{0.0, 0u, 0u};
  return true;
}

// ------------------------------------------------------------------ overlay records (fast mode)
// PSI[b, a] departs from init_prefs[a] only where (b, a) was backed up (tree.py:247-253,
// backup.py:107-108).  In fast mode a belief's row is therefore the initial row overlaid with
// its realised cells, kept inline in a 32-B record (one sector) -- child k of b owns slot k --
// and only a belief with more than kOverlay action children gets a dense row (allocated from
// its own pool, so PSI memory scales with the busy beliefs, not with every belief).  The
// search reads records; the backup writes their cells; a dense row is written by the search
// lane that creates the (kOverlay + 1)-th child and is used from the next pass on.
constexpr int kOverlay = VP_OVERLAY_SLOTS;
template <class PsiT>
struct __align__(16) Rec {
  u32 dense_pass;                // 0: no dense row; else the pass whose search wrote it
  u32 dense_row;                 // row of T.psi
  unsigned short act[kOverlay];  // action + 1; 0 = empty slot
  PsiT val[kOverlay];            // PSI[b, act - 1]
};
static_assert(sizeof(Rec<float>) == 32 && sizeof(Rec<double>) == 48, "overlay record layout (vpb200.h)");

template <class PsiT>
__device__ __forceinline__ Rec<PsiT>* rec_ptr(const vp_tree& T, int b) {
  return reinterpret_cast<Rec<PsiT>*>(T.b_rec) + b;
}
template <class PsiT, bool L2 = false>
__device__ __forceinline__ Rec<PsiT> load_rec(const vp_tree& T, int b) {
  const uint4* p = reinterpret_cast<const uint4*>(rec_ptr<PsiT>(T, b));
  Rec<PsiT> r;
  uint4* q = reinterpret_cast<uint4*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Rec<PsiT>) / 16); ++i) q[i] = L2 ? __ldcg(p + i) : p[i];
  return r;
}
// Per dense row: the LSE and pass of the backup that last changed it (CDF rebuild requests).
struct __align__(16) DenseMeta {
  double lse;
  u32 pass;
  u32 pad;
};

// The dense PSI row of belief b, or -1 while it keeps an overlay record (one 8-B load).
template <class PsiT>
__device__ __forceinline__ int dense_row_of(const vp_tree& T, int b) {
  const uint2 w = *reinterpret_cast<const uint2*>(rec_ptr<PsiT>(T, b));
  return w.x ? (int)w.y : -1;
}
template <class PsiT>
__device__ __forceinline__ bool rec_any(const Rec<PsiT>& r) {
  u32 any = 0;
#pragma unroll
  for (int k = 0; k < kOverlay; ++k) any |= r.act[k];
  return any != 0;
}

// log(exp(a) + exp(b)) without overflow / underflow (fp64)
__device__ __forceinline__ double log_add_exp(double a, double b) {
  const double hi = a > b ? a : b, lo = a > b ? b : a;
  return lo == -INFINITY ? hi : hi + log1p(exp(lo - hi));
}

// Delivery of a log-mass to an overlay belief (fast mode, at most kOverlay deliveries per pass:
// one per action child): the accumulator's sum holds log sum exp of the delivered log-masses,
// combined by CAS (an empty accumulator has rows == 0; every delivery carries >= 1 row).
__device__ __forceinline__ bool acc_deliver_log(void* base, int i, double l, u32 drows, u32 dcnt, u32 target,
                                                Acc& out) {
  if ((drows & kRowsMask) == target) {
    out = Acc{l, drows, dcnt};
    return true;
  }
  Acc* p = reinterpret_cast<Acc*>(base) + i;
  u64 lo = 0, hi = 0;
  while (true) {
    const double s = hi == 0 ? l : log_add_exp(__longlong_as_double((long long)lo), l);
    const u32 r = (u32)hi + drows, c = (u32)(hi >> 32) + dcnt;
    const u64 nlo = (u64)__double_as_longlong(s), nhi = (u64)r | ((u64)c << 32);
    u64 olo, ohi;
    cas128(p, lo, hi, nlo, nhi, olo, ohi);
    if (olo == lo && ohi == hi) {
      if ((r & kRowsMask) != target) return false;
      out = Acc{s, r, c};
      *p = Acc{0.0, 0u, 0u};
      return true;
    }
    lo = olo;
    hi = ohi;
  }
}

// ------------------------------------------------------------------ exp helpers (fast mode)
// exp(eta * psi - shift) is evaluated as exp2(fma(eta*log2e, psi, -shift*log2e)).
// fp32: one MUFU.EX2 (flush-to-zero: probabilities below 2^-126 are zero mass)
__device__ __forceinline__ float fexp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double fexp2(double x) { return exp2(x); }
__device__ __forceinline__ float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double ffma(double a, double b, double c) { return __fma_rn(a, b, c); }
constexpr double kLog2eD = 1.4426950408889634;

// Loads of PSI: plain (search: rows are stable for the whole kernel) or L2
// (backup: rows are rewritten by other SMs inside the kernel).
template <bool L2, class T>
__device__ __forceinline__ T ldp(const T* p) {
  if constexpr (L2) return __ldcg(p);
  else return *p;
}

// ------------------------------------------------------------------ LSE

__device__ __forceinline__ double lse_log(float s) { return (double)logf(s); }
__device__ __forceinline__ double lse_log(double s) { return log(s); }

// Fast LSE (backup.py:34-41 formula: max, then sum of exp) by a group of G
// lanes per row with the row held in registers, so short rows (|A| <= 16 G)
// keep every lane busy and take one memory round trip.  All 32 lanes must
// call it (rows may be null for idle groups).
__host__ __device__ constexpr int lse_group_size(int A) {
  return A <= 16 ? 1 : A <= 32 ? 2 : A <= 64 ? 4 : A <= 128 ? 8 : A <= 256 ? 16 : 32;
}

template <class PsiT, int G, bool L2 = false>
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
      v[k] = (row && a < A) ? ldp<L2>(row + a) : -(PsiT)INFINITY;
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
        const PsiT z = e * ldp<L2>(row + a);
        m = z > m ? z : m;
      }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const PsiT w = __shfl_xor_sync(FULL, m, o, G);
      m = w > m ? w : m;
    }
    const PsiT m2 = m * (PsiT)kLog2eD;
    if (row)
      for (int a = gl; a < A; a += G) s += fexp2(ffma(e2, ldp<L2>(row + a), -m2));
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

// Streaming log-sum-exp of the elements start, start + stride, ... of an L2-resident row in fp64:
// mx = max eta psi, sm = sum exp(eta psi - mx) over them.  Batches of 8 independent loads, the
// running sum rescaled once per batch.
template <class PsiT>
__device__ __forceinline__ void lse_online_f64(const PsiT* r, int A, int start, int stride, double eta, double& mx,
                                               double& sm) {
  for (int a0 = start; a0 < A; a0 += 8 * stride) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int a = a0 + j * stride;
      v[j] = a < A ? eta * (double)__ldcg(r + a) : -INFINITY;
    }
    double mb = v[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) mb = fmax(mb, v[j]);
    const double mn = fmax(mx, mb);
    double acc = mx == -INFINITY ? 0.0 : sm * exp(mx - mn);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j] == -INFINITY ? 0.0 : exp(v[j] - mn);
    sm = acc;
    mx = mn;
  }
}

// LSE of a row in fp64 arithmetic by a full warp (returned on every lane).  Fast mode keeps
// every cached LSE at fp64 accuracy whatever the PSI dtype: the incremental backup LSE
// (1 + sum of changed terms) cancels terms of order 1, so LSE_pre must not carry the
// ~1e-7 error of an fp32 evaluation.
template <class PsiT, bool L2 = false>
__device__ double row_lse_f64(const PsiT* row, int A, double eta) {
  double m = -INFINITY;
  for (int a = lane_id(); a < A; a += 32) m = fmax(m, eta * (double)ldp<L2>(row + a));
  m = warp_max(m);
  double s = 0.0;
  for (int a = lane_id(); a < A; a += 32) s += exp(eta * (double)ldp<L2>(row + a) - m);
  s = warp_sum(s);
  return m / eta + log(s) / eta;
}

// numpy-order LSE for the fp64 parity mode: m/eta + log(pairwise sum)/eta.
template <bool L2 = false>
__device__ double lse_exact(const double* row, int A, double eta) {
  double m = -INFINITY;
  for (int a = 0; a < A; ++a) m = fmax(m, eta * ldp<L2>(row + a));
  auto ex = [&](int a) -> double { return exp(eta * ldp<L2>(row + a) - m); };
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
__device__ __forceinline__ int search_cdf(const CT* cdf, int A, CT u) {
  int lo = 0, hi = A;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cdf[mid] > u) hi = mid;
    else lo = mid + 1;
  }
  return lo < A ? lo : A - 1;
}

// Draw from an overlay row (search.py:46-83 on init + realised cells): with the row's LSE,
//   F(a) = s * initCDF(a) + sum_{k: a_k <= a} c_k,   s = exp(eta (LSE_init - LSE)),
//   c_k = exp(eta (psi_k - LSE)) - exp(eta (init_{a_k} - LSE)),
// is the row's CDF (the initial CDF rescaled, each realised cell's mass swapped in); the
// first a with F(a) > u, clamped to |A| - 1.  Probabilities use the dense sampler's
// arithmetic (exp2(fma(eta log2e, psi, -eta LSE log2e))).
template <class PsiT>
__device__ __forceinline__ int draw_overlay(const Rec<PsiT>& r, const PsiT* init_cdf, const PsiT* init_row, int A,
                                            double eta, double lse, double lse_init, PsiT u) {
  const PsiT e2 = (PsiT)(eta * kLog2eD), sh2 = (PsiT)(eta * lse * kLog2eD);
  const PsiT s = (PsiT)exp(eta * (lse_init - lse));
  int ak[kOverlay];
  PsiT ck[kOverlay];
#pragma unroll
  for (int k = 0; k < kOverlay; ++k) {
    ak[k] = r.act[k] ? (int)r.act[k] - 1 : A;
    ck[k] = r.act[k] ? fexp2(ffma(e2, r.val[k], -sh2)) - fexp2(ffma(e2, init_row[ak[k]], -sh2)) : (PsiT)0;
  }
  int lo = 0, hi = A;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    PsiT f = s * init_cdf[mid];
#pragma unroll
    for (int k = 0; k < kOverlay; ++k) f += ak[k] <= mid ? ck[k] : (PsiT)0;
    if (f > u) hi = mid;
    else lo = mid + 1;
  }
  return lo < A ? lo : A - 1;
}

// A staged PSI row (shared memory) becomes its unnormalised CDF, in place:
// lane j owns the contiguous columns [j C, j C + C), C = ceil(A / 32), keeps a
// running sum over them, and one warp scan adds the preceding lanes' totals.
// Returns the row total (the softmax normaliser) on every lane.
template <class PsiT>
struct VecOf;
template <>
struct VecOf<float> {
  typedef float4 T;
  static constexpr int N = 4;
};
template <>
struct VecOf<double> {
  typedef double2 T;
  static constexpr int N = 2;
};
template <class PsiT, bool Normalise = false>
__device__ __forceinline__ PsiT row_cdf_inplace(PsiT* row, int A, PsiT e2, PsiT sh2) {
  typedef VecOf<PsiT> V;
  const int C = (A + 31) >> 5;
  const int lo = lane_id() * C, hi = min(A, lo + C);
  PsiT loc = 0;
  const bool vec = (C % V::N) == 0;  // chunks start 16-B aligned: vector LDS/STS
  if (vec) {
    for (int c = lo; c < hi; c += V::N) {
      typename V::T v = *reinterpret_cast<typename V::T*>(row + c);
      PsiT* x = reinterpret_cast<PsiT*>(&v);
#pragma unroll
      for (int j = 0; j < V::N; ++j) {
        loc += (c + j < hi) ? fexp2(ffma(e2, x[j], -sh2)) : (PsiT)0;
        x[j] = loc;
      }
      *reinterpret_cast<typename V::T*>(row + c) = v;
    }
  } else {
    for (int c = lo; c < hi; ++c) {
      loc += fexp2(ffma(e2, row[c], -sh2));
      row[c] = loc;
    }
  }
  const PsiT incl = warp_inclusive_scan(loc);
  const PsiT up = __shfl_up_sync(FULL, incl, 1);  // all 32 lanes take part in the shuffle
  const PsiT excl = lane_id() ? up : (PsiT)0;
  const PsiT total = __shfl_sync(FULL, incl, 31);
  if (Normalise || lane_id() > 0) {
    const PsiT scale = Normalise ? (PsiT)1 / total : (PsiT)1;
    if (vec) {
      for (int c = lo; c < hi; c += V::N) {
        typename V::T v = *reinterpret_cast<typename V::T*>(row + c);
        PsiT* x = reinterpret_cast<PsiT*>(&v);
#pragma unroll
        for (int j = 0; j < V::N; ++j) x[j] = Normalise ? (x[j] + excl) * scale : x[j] + excl;
        *reinterpret_cast<typename V::T*>(row + c) = v;
      }
    } else {
      for (int c = lo; c < hi; ++c) row[c] = Normalise ? (row[c] + excl) * scale : row[c] + excl;
    }
  }
  __syncwarp();
  return total;
}

// The normalised softmax CDF of a PSI row into global memory (search.py:46-54, 77-79):
// p_a = exp(eta (psi_a - lse)), running sums divided by their total.  A full warp; lane j owns
// the contiguous columns [j C, j C + C), C = ceil(|A| / 32), and the row is read twice (total,
// then the stored sums), so any |A| fits without staging.  L2: the row was written by other
// SMs inside this kernel.
template <class PsiT, bool L2>
__device__ void build_cdf_row(const PsiT* row, PsiT* cdf, int A, double eta, double lse) {
  const PsiT e2 = (PsiT)(eta * kLog2eD), sh2 = (PsiT)(eta * lse * kLog2eD);
  const int C = (A + 31) >> 5;
  const int lo = lane_id() * C, hi = min(A, lo + C);
  constexpr int R = 16;
  if (C <= R) {  // |A| <= 512: the lane's chunk in registers, all its loads in flight at once
    PsiT v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = lo + j < hi ? ldp<L2>(row + lo + j) : (PsiT)0;
    PsiT loc = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      loc += lo + j < hi ? fexp2(ffma(e2, v[j], -sh2)) : (PsiT)0;
      v[j] = loc;
    }
    const PsiT incl = warp_inclusive_scan(loc);
    const PsiT up = __shfl_up_sync(FULL, incl, 1);
    const PsiT excl = lane_id() ? up : (PsiT)0;
    const PsiT scale = (PsiT)1 / __shfl_sync(FULL, incl, 31);
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (lo + j < hi) cdf[lo + j] = (v[j] + excl) * scale;
    return;
  }
  PsiT loc = 0;
  for (int c = lo; c < hi; ++c) loc += fexp2(ffma(e2, ldp<L2>(row + c), -sh2));
  const PsiT incl = warp_inclusive_scan(loc);
  const PsiT up = __shfl_up_sync(FULL, incl, 1);
  const PsiT excl = lane_id() ? up : (PsiT)0;
  const PsiT scale = (PsiT)1 / __shfl_sync(FULL, incl, 31);
  loc = 0;
  for (int c = lo; c < hi; ++c) {
    loc += fexp2(ffma(e2, ldp<L2>(row + c), -sh2));
    cdf[c] = (loc + excl) * scale;
  }
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
  int rows;    // PSI rows staged per warp per batch
  int stride;  // staged row stride in PsiT elements (odd multiple of 16 bytes)
};

// Per-warp staging state (buffer, mbarrier, phase parity).
template <class PsiT>
struct Stage {
  PsiT* buf;
  u64* bar;
  u32 phase;
  StageCfg cfg;
};

// ------------------------------------------------------------------ warp helpers

// Sum of v over the lanes in `grp`, in lane (= row) order, delivered to all
// lanes; as many shuffle rounds as the largest group has members.
__device__ __forceinline__ double group_sum_ordered(double v, u32 grp) {
  const int rounds = (int)__reduce_max_sync(FULL, (unsigned)__popc(grp));
  u32 m = grp;
  double s = 0.0;
  for (int t = 0; t < rounds; ++t) {
    const double x = __shfl_sync(FULL, v, m ? __ffs(m) - 1 : lane_id());
    if (m) {
      s += x;
      m &= m - 1u;
    }
  }
  return s;
}
// Same, short-circuited when every active key of the warp is distinct.
__device__ __forceinline__ double group_sum(double v, u32 grp, bool active) {
  if (__all_sync(FULL, !active || __popc(grp) == 1)) return v;
  return group_sum_ordered(v, grp);
}

// Write the initial PSI row (tree.py:253) into the rows named by the lanes
// set in `mask` (lazy rows become real the first time they are interior):
// each such lane issues ONE TMA bulk store of the block's shared copy of the
// initial row; the copy engine moves the bytes, the warp moves on.  Rows are
// only read after this kernel (or as staged rows of non-lazy beliefs), and
// bulk_store_drain() at the end of the warp's work completes the stores.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, u32 bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_store_drain() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class PsiT>
__device__ __forceinline__ void materialise_rows(const vp_tree& T, const PsiT* init_row, u32 mask, int b) {
  if (!((mask >> lane_id()) & 1u)) return;
  PsiT* psi = reinterpret_cast<PsiT*>(T.psi);
  const u32 bytes = (u32)(((size_t)T.action_count * sizeof(PsiT) + 15) & ~(size_t)15);
  bulk_s2g(psi + (size_t)b * T.psi_stride, init_row, bytes);
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Fast mode: belief b just got its (kOverlay + 1)-th action child -- give it a dense row:
// the initial row (one TMA bulk store from the block's shared copy) with the record's
// realised cells written over it (stable during the search: only the backup writes them),
// then publish {row, pass}.  Draws of this pass keep using the record (dense_pass == pass).
template <class PsiT>
__device__ __noinline__ void materialise_dense(const vp_tree& T, unsigned long long* stats, int b,
                                               const Rec<PsiT>& rec, const PsiT* init_row, u32 pass) {
  const int r = atomicAdd(&T.counters[VP_COUNTER_DENSE], 1);
  if (r >= T.cap_dense) {
    T.counters[2] = 1;  // overflow: the host fails the plan loudly
    return;
  }
  PsiT* row = reinterpret_cast<PsiT*>(T.psi) + (size_t)r * T.psi_stride;
  const u32 bytes = (u32)(((size_t)T.action_count * sizeof(PsiT) + 15) & ~(size_t)15);
  if (init_row) {
    bulk_s2g(row, init_row, bytes);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
  } else {
    for (int a = 0; a < T.action_count; ++a) row[a] = (PsiT)T.init_prefs[a];
  }
#pragma unroll
  for (int k = 0; k < kOverlay; ++k)
    if (rec.act[k]) row[rec.act[k] - 1] = rec.val[k];
  Rec<PsiT>* g = rec_ptr<PsiT>(T, b);
  g->dense_row = (u32)r;
  g->dense_pass = pass;
  if (stats) atomicAdd(&stats[10], 1ull);
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
      v = __shfl_sync(FULL, v, 0);
    } else {
      v = row_lse_f64<PsiT>(psi, A, T.eta);
    }
    // normalised CDF of the initial row with the fast sampler's arithmetic (warp-parallel)
    PsiT* cdf = reinterpret_cast<PsiT*>(T.init_cdf);
    for (int a = threadIdx.x; a < A; a += 32) cdf[a] = psi[a];
    __syncwarp();
    const PsiT total = row_cdf_inplace(cdf, A, (PsiT)(T.eta * kLog2eD), (PsiT)(T.eta * v * kLog2eD));
    for (int a = threadIdx.x; a < A; a += 32) cdf[a] = cdf[a] / total;
    if constexpr (!Exact)  // the root's dense row 0 is the initial row: its CDF row too
      build_cdf_row<PsiT, false>(psi, reinterpret_cast<PsiT*>(T.psi_cdf), A, T.eta, v);
    if (threadIdx.x == 0) {
      T.init_lse[0] = v;
      T.b_lse[0] = v;
      T.b_parent_action[0] = -1;
      T.b_parent_obs[0] = 0xffffffffu;
      T.b_parent_belief[0] = -1;
      T.b_parent_act[0] = -1;
      T.b_depth[0] = 0;
      T.b_value[0] = 0.0;
      T.b_rows[0] = 0;
      reinterpret_cast<Acc*>(T.b_acc)[0] = Acc{0.0, 0u, 0u};
      T.b_flags[0] = 0;  // the root row is written (above), not lazy
      T.b_ckey[0] = 0;
      T.b_nact[0] = 0;
      if constexpr (!Exact) {  // the root owns dense row 0 from the start (it is the busiest row)
        Rec<PsiT> r{};
        r.dense_pass = 1;
        r.dense_row = 0;
        *rec_ptr<PsiT>(T, 0) = r;
        T.counters[VP_COUNTER_DENSE] = 1;
      }
      T.counters[0] = 1;
      T.counters[VP_COUNTER_ACTIONS] = 0;
      T.counters[VP_COUNTER_LIVE_B] = 1;
      T.counters[VP_COUNTER_LIVE_A] = 0;
      T.counters[VP_COUNTER_DONE] = 0;
      T.counters[2] = 0;
      T.counters[3] = 0;
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ root-state draw

// belief.py:37-44: u = uniform(draw_key, row); first index with cum > u
// (searchsorted side=right), clamped to m - 1.
__device__ __forceinline__ int draw_index(const double* cumw, int m, u64 key, int r, int rk) {
  const double u = uniform1(key, (u64)r, rk);
  // weights are uniform after every SIR update (belief.py:101): the first
  // guess floor(u m) is usually the answer, confirmed with two loads
  int idx = min((int)(u * (double)m), m - 1);
  const double hi_v = cumw[idx], lo_v = idx ? cumw[idx - 1] : -1.0;
  if (!(hi_v > u && lo_v <= u)) {
    int lo = 0, hi = m;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cumw[mid] > u) hi = mid;
      else lo = mid + 1;
    }
    idx = lo < m - 1 ? lo : m - 1;
  }
  return idx;
}

template <class State>
__device__ __forceinline__ State draw_state(const State* particles, const double* cumw, int m, u64 key, int r,
                                             int rk) {
  return particles[draw_index(cumw, m, key, r, rk)];
}

// ------------------------------------------------------------------ cooperative models
// A model whose record is too large for one lane (CrowdNav) declares kCoop: the
// search then carries ONE row per warp, keeps its record in shared memory and
// calls Model::step_warp with all 32 lanes, which split the work inside the row.
template <class M, class = void>
struct coop_trait : std::false_type {};
template <class M>
struct coop_trait<M, std::void_t<decltype(M::kCoop)>> : std::integral_constant<bool, M::kCoop> {};
// (insert replays recorded trajectories without stepping the model: full warps)
template <class Model>
__host__ __device__ constexpr int rows_per_search_warp(int mode, int rows = 32) {
  return coop_trait<Model>::value && mode != VP_SEARCH_INSERT ? 1 : rows;
}

struct NoState {};
template <class State>
__device__ __forceinline__ State& state_slot(State* shared, NoState&) { return *shared; }
template <class State>
__device__ __forceinline__ State& state_slot(State*, State& local) { return local; }

// whole-warp copy of one record (8-byte words; records are 8-byte aligned)
template <class State>
__device__ __forceinline__ void warp_copy_state(State& dst, const State& src) {
  static_assert(sizeof(State) % 8 == 0, "records are whole 8-byte words");
  u64* d = reinterpret_cast<u64*>(&dst);
  const u64* q = reinterpret_cast<const u64*>(&src);
  for (int i = lane_id(); i < (int)(sizeof(State) / 8); i += 32) d[i] = q[i];
  __syncwarp();
}

// one generative step of every live row of the warp (search.py:113-115)
// RK: the stream kind (vp_rng_kind) as a compile-time constant of the search kernel
template <class Model, int RK>
__device__ __forceinline__ void model_step(const vp_model& M, typename Model::State& st, int a, u64 key, int rg,
                                           bool live, u32& o, double& rw) {
  if constexpr (coop_trait<Model>::value) {
    // the row is lane 0's; every lane takes part
    Model::step_warp(M, st, __shfl_sync(FULL, a, 0), key, (u64)__shfl_sync(FULL, rg, 0),
                     __shfl_sync(FULL, (int)live, 0) != 0, o, rw, RK);
  } else if (live) {
    Model::step(M, st, a, key, (u64)rg, o, rw, RK);
  }
}

// ------------------------------------------------------------------ search

// Softmax draw of one action per lane (search.py:46-83) from the PSI row of belief b.  Called by
// all 32 lanes; lanes with ok == false return 0.
//  * parity mode: numpy-order inverse CDF of the row (the initial row while lazily initial);
//  * fast mode: a belief with an overlay record draws from the shared initial CDF corrected by
//    its realised cells; a belief with a dense row draws from that row's CDF, which the backup
//    that last changed the row rebuilt (PSI is read-only during a pass): the warp's distinct
//    dense beliefs get ONE TMA bulk copy each into the warp's stage, then every lane
//    binary-searches its row.
template <class PsiT, bool Exact>
__device__ __forceinline__ int draw_action(const vp_tree& T, const vp_work& W, Stage<PsiT>& sg, const PsiT* init_cdf,
                                           const PsiT* init_row, int b, u32 fl, const Rec<PsiT>& rec, double lse,
                                           double lse_init, bool ok, double u, u32 pass) {
  const int A = T.action_count, lane = lane_id();
  int a = 0;
  if constexpr (Exact) {
    if (ok) {
      const double* row =
          (fl & 1u) ? T.init_prefs : reinterpret_cast<const double*>(T.psi) + (size_t)b * T.psi_stride;
      a = sample_exact(row, A, T.eta, u);
    }
  } else {
    VP_DR_INIT();
    // a dense row written before this pass (one written during it is used from the next pass)
    const bool need = ok && rec.dense_pass != 0 && rec.dense_pass < pass;
    const bool ovl = ok && !need && rec_any(rec);
    if (ok && !need)
      a = ovl ? draw_overlay<PsiT>(rec, init_cdf, init_row, A, T.eta, lse, lse_init, (PsiT)u)
              : search_cdf(init_cdf, A, (PsiT)u);
    if (W.stats) {
      const u32 om = __ballot_sync(FULL, ovl);
      if (lane == 0 && om) atomicAdd(&W.stats[9], (unsigned long long)__popc(om));
    }
    VP_DR(1);
    const u32 g = __match_any_sync(FULL, need ? (u32)b : 0xffffffffu);
    const int my_leader = __ffs(g) - 1;
    const bool lead = need && lane == my_leader;
    const u32 leaders = __ballot_sync(FULL, lead);
    const int K = __popc(leaders);
    if (W.stats && lane == 0 && K) atomicAdd(&W.stats[2], (unsigned long long)K);
    const int my_slot = need ? __popc(leaders & ((1u << my_leader) - 1u)) : -1;
    const PsiT* cdf = reinterpret_cast<const PsiT*>(T.psi_cdf);
    const u32 row_bytes = (u32)(((size_t)A * sizeof(PsiT) + 15) & ~(size_t)15);
    for (int s0 = 0; s0 < K; s0 += sg.cfg.rows) {
      const int cnt = min(sg.cfg.rows, K - s0);
      fence_async_smem();  // the stage's previous rows were read by the generic proxy
      if (lane == 0) mbar_expect_tx(sg.bar, row_bytes * (u32)cnt);
      __syncwarp();
      const bool mine = need && my_slot >= s0 && my_slot < s0 + cnt;
      const PsiT* srow = sg.buf + (size_t)(my_slot - s0) * sg.cfg.stride;
      if (mine && lane == my_leader)
        bulk_g2s(const_cast<PsiT*>(srow), cdf + (size_t)rec.dense_row * T.psi_stride, row_bytes, sg.bar);
      VP_DR(3);
      mbar_wait(sg.bar, sg.phase);
      sg.phase ^= 1u;
      VP_DR(4);
      if (mine) a = search_cdf(srow, A, (PsiT)u);
      __syncwarp();
      VP_DR(6);
    }
  }
  return a;
}


// Rows arriving at belief c (one reduction per distinct belief of the warp).
// At the leaf level the first arrival also appends c to the leaf list (one
// list atomic per warp).  Called by all lanes.
__device__ __forceinline__ void arrive(const vp_tree& T, const vp_work& W, int* leaf_count, int c, u32 grp,
                                       bool lead, bool leaf_level) {
  const int cnt = __popc(grp);
  if (!leaf_level) {
    if (lead) red_add(&T.b_rows[c], cnt);
    return;
  }
  const bool first = lead && atomicAdd(&T.b_rows[c], cnt) == 0;
  const u32 fm = __ballot_sync(FULL, first);
  if (!fm) return;
  const int src = __ffs(fm) - 1;
  int base = 0;
  if (lane_id() == src) base = atomicAdd(leaf_count, __popc(fm));
  base = __shfl_sync(FULL, base, src);
  if (first) W.leaves[base + __popc(fm & ((1u << lane_id()) - 1u))] = c;
}

// Read-only probe of a hash index (no inserts run concurrently): node id or -1.
__device__ __forceinline__ int find_key(const Slot* tab, u64 mask, u64 key) {
  u64 h = slot_hash(key) & mask;
  while (true) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(tab + h));
    if (v.x == key) return (int)(u32)v.y;
    if (v.x == kEmptyKey) return -1;
    h = (h + 1) & mask;
  }
}

// VP_SEARCH_TRAJECTORY: the rows' actions, observations, rewards and leaf
// values against the tree as it stands (no node is created).  A row whose path
// leaves the existing tree draws from the initial row from then on -- exactly
// what the fused search does, since nodes created during a pass are lazily
// initial -- so the trajectory is that of the fused search.
template <class Model, class PsiT, bool Exact, int RK>
__device__ void trajectory_rows(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_search_args& S,
                                Stage<PsiT>& sg, const PsiT* init_cdf, const PsiT* init_row, double lse_init,
                                typename Model::State& st, int r, int rg, bool active, u64 skey) {
  const int n = W.n;
  const Slot* ha = slots(T.hash_a);
  const Slot* hb = slots(T.hash_b);
  int b = 0;
  bool known = active;  // the row's belief existed when the pass started
  u32 fl = known ? T.b_flags[0] : 1u;
  Rec<PsiT> rec{};  // fast mode: the belief's overlay record (zero: initial row)
  double lse = lse_init;
  if constexpr (!Exact) {
    if (known) {
      rec = load_rec<PsiT>(T, 0);
      lse = T.b_lse[0];
    }
  }
  for (int l = 0; l < S.d_max; ++l) {
    const u64 lkey = fold(skey, (u64)l);
    const double u = active ? uniform1(fold(lkey, 0), (u64)rg, RK) : 0.0;
    const int a = draw_action<PsiT, Exact>(T, W, sg, init_cdf, init_row, b, known ? fl : 1u, rec, lse, lse_init, active,
                                           u, S.pass);
    u32 o = 0;
    double rw = 0.0;
    model_step<Model, RK>(M, st, a, fold(lkey, 1), rg, active, o, rw);
    if (active) {
      const size_t t = (size_t)l * n + r;
      W.trace_action[t] = a;
      W.trace_obs[t] = o;
      W.trace_reward[t] = rw;
    }
    if (known) {
      const int x = find_key(ha, T.hmask_a, ((u64)(u32)b << 32) | (u32)a);
      const int c = x < 0 ? -1 : find_key(hb, T.hmask_b, belief_key(T, b, a, x, o));
      known = c >= 0;
      if (known) {
        b = c;
        fl = T.b_flags[c];
        if constexpr (!Exact) {
          rec = load_rec<PsiT>(T, c);
          lse = T.b_lse[c];
        }
      } else if constexpr (!Exact) {
        rec = Rec<PsiT>{};  // off the tree: the initial row from here on
        lse = lse_init;
      }
    }
  }
  if (active) W.leaf_value[r] = Model::heuristic(M, st);
}

// The search kernel body for one warp = 32 consecutive rows.
template <class Model, class PsiT, bool Exact, int RK>
__device__ void search_warp(const vp_tree& T, const vp_model& M, const vp_work& W, const vp_search_args& S,
                            Stage<PsiT>& sg, const PsiT* init_cdf, const PsiT* init_row, int warp_index,
                            typename Model::State* shared_state, int rows, int base_a, int base_b) {
  typedef typename Model::State State;
  constexpr bool kCoop = coop_trait<Model>::value;
  const int kRows = rows_per_search_warp<Model>(S.mode, rows);
  const int n = W.n, lane = lane_id();
  // 32 rows per warp: rows of a warp at the same belief share one draw (match_any
  // groups), which pays more than the latency hiding of more, emptier warps
  // (16 rows per warp: +27 % search time at C2).  Cooperative models: one row.
  const int r = lane < kRows ? warp_index * kRows + lane : n;
  const int rg = S.row0 + r;  // global row id: RNG streams and creation keys
  const bool active = r < n;
  const bool insert = S.mode == VP_SEARCH_INSERT;
  const int d = S.d_max, depth0 = S.depth0;
  const u32 pass = S.pass;
  const u64 skey = S.search_key_dev ? *S.search_key_dev : S.search_key;
  Slot* ha = slots(T.hash_a);
  Slot* hb = slots(T.hash_b);
  int* leaf_count = W.leaf_count + (pass & 1u);

  typename std::conditional<kCoop, NoState, State>::type own{};
  State& st = state_slot<State>(shared_state, own);
  if constexpr (kCoop) {
    if (!insert) {  // lane 0 picks the record, the warp copies it into shared memory
      const State* src = nullptr;
      if (active) {
        const u64 dkey = S.draw_key_dev ? *S.draw_key_dev : S.draw_key;
        src = S.particles ? reinterpret_cast<const State*>(S.particles) +
                                draw_index(S.cum_weights, S.m, dkey, rg, RK)
                          : reinterpret_cast<const State*>(W.states) + r;
      }
      src = reinterpret_cast<const State*>(__shfl_sync(FULL, (unsigned long long)src, 0));
      if (src) warp_copy_state(st, *src);
    }
  } else if (active && !insert) {
    if (S.particles) {
      const u64 dkey = S.draw_key_dev ? *S.draw_key_dev : S.draw_key;
      st = draw_state(reinterpret_cast<const State*>(S.particles), S.cum_weights, S.m, dkey, rg, RK);
    } else {
      st = reinterpret_cast<const State*>(W.states)[r];
    }
  }
  if (S.mode == VP_SEARCH_TRAJECTORY) {
    trajectory_rows<Model, PsiT, Exact, RK>(T, M, W, S, sg, init_cdf, init_row, T.init_lse[0], st, r, rg, active, skey);
    return;
  }
  int b = active ? (S.start_beliefs ? S.start_beliefs[r] : 0) : 0;
  bool ok = active;
  u32 fl = Exact && ok ? T.b_flags[b] : 0u;  // flags of nodes older than this pass are stable here
  // fast mode: the lane's view of its belief -- overlay record and cached LSE (stable during
  // the search except a dense row's publication, which draws of this pass ignore)
  const double lse_init = T.init_lse[0];
  Rec<PsiT> rec{};
  double lse = lse_init;
  if constexpr (!Exact) {
    if (ok) {
      rec = load_rec<PsiT>(T, b);
      lse = T.b_lse[b];
    }
  }
  u32 grp = __match_any_sync(FULL, ok ? (u32)b : 0xffffffffu);
  bool lead = ok && lane == __ffs(grp) - 1;
  arrive(T, W, leaf_count, b, grp, lead, depth0 == d);

  // An interior frontier (depth0 > 0): the rows also count toward every
  // ancestor, so the completion wave of the backup reaches the root
  // (backup.py:90-95 derives those levels from the valued children).
  if (depth0 > 0 && S.start_beliefs) {
    int cur = b;
    for (int k = depth0; k > 0; --k) {
      const int x = ok ? T.b_parent_action[cur] : -1;
      const u32 g = __match_any_sync(FULL, (u32)x);
      const bool ld = ok && lane == __ffs(g) - 1;
      const int p = ok ? T.a_parent_belief[x] : 0;
      bool mat = false;
      if (ld) {
        red_add(&T.a_rows[x], __popc(g));
        red_add(&T.b_rows[p], __popc(g));
        if (Exact && (T.b_flags[p] & 2u)) mat = atomicAnd(&T.b_flags[p], ~2u) & 2u;
      }
      if constexpr (Exact) materialise_rows<PsiT>(T, init_row, __ballot_sync(FULL, mat), p);
      cur = p;
    }
  }

  bool made_interior = false;  // this lane created b at the previous level and it is interior now
  // fast mode: the action this lane created at the previous level (its overlay slot is stored
  // one level later) and a belief owed a dense row (written after the levels)
  int pend_x = -1, pend_k = 0, pend_bel = -1, pend_mat = -1, pend_mat_prev = -1;
  int won_a = 0, won_b = 0;    // nodes this lane created (live counts, one reduction per warp)
  VP_PH_INIT();
  for (int l = depth0; l < d; ++l) {
    const u64 lkey = fold(skey, (u64)l);  // search.py:107
    // ---- parity mode, lazy rows: b is interior at this level; write its PSI row once
    if constexpr (Exact) {
      bool mat = made_interior;
      if (lead && !made_interior && (fl & 2u)) mat = atomicAnd(&T.b_flags[b], ~2u) & 2u;
      materialise_rows<PsiT>(T, init_row, __ballot_sync(FULL, mat), b);
    }
#ifdef VP_PHASE_CLOCKS
    { u32 w_; asm volatile("mov.b32 %0, %1;" : "=r"(w_) : "r"(rec.dense_pass)); (void)w_; }
    VP_PH(0);
#endif
    // ---- softmax draw (search.py:108-112)
    const double u = (active && !S.inject_actions) ? uniform1(fold(lkey, 0), (u64)rg, RK) : 0.0;  // level_rng.derive(0)
    int a = 0;
    if (S.inject_actions) a = active ? S.inject_actions[(size_t)l * n + r] : 0;
    else a = draw_action<PsiT, Exact>(T, W, sg, init_cdf, init_row, b, fl, rec, lse, lse_init, ok, u, pass);
    // ---- generative model (search.py:113-115), state stays in registers
    u32 o = 0;
    double rw = 0.0;
    if (insert) {
      if (active) {
        o = S.inject_obs[(size_t)l * n + r];
        rw = S.inject_reward[(size_t)l * n + r];
      }
    } else {
      VP_PH(1);
      model_step<Model, RK>(M, st, a, fold(lkey, 1), rg, ok, o, rw);  // level_rng.derive(1)
      VP_PH(2);
    }

    // ---- action node (b, a) and belief node: append_actions / append_beliefs (tree.py:180-256)
    // Ids are static: row r creating at this level takes extent + (l - depth0) n + r in each
    // table, so a claim is ONE 128-bit CAS that inserts {key, pass | id} -- no id atomic, no
    // publication, no spinning on another row's claim.  With (belief, action, obs) belief keys
    // (bkey_mode 1) the two claims of a level are in flight together.
    const bool early = T.bkey_mode != 0;
    const bool interior_next = l + 1 < d;
    const long long id_off = (long long)(l - depth0) * n + r;
    const long long my_a = (long long)base_a + id_off, my_b = (long long)base_b + id_off;
    const u64 key_a = ((u64)(u32)b << 32) | (u32)a;
    const u32 grp_a = __match_any_sync(FULL, ok ? key_a : kEmptyKey);
    const int leader_a = __ffs(grp_a) - 1;
    bool lead_a = ok && lane == leader_a;
    u64 key_b = early ? belief_key(T, b, a, 0, o) : 0ull;
    u32 grp_b = early ? __match_any_sync(FULL, ok ? key_b : kEmptyKey) : 0u;
    int leader_b = early ? __ffs(grp_b) - 1 : 0;
    bool lead_b = early && ok && lane == leader_b;
    if ((lead_a && my_a >= T.cap_actions) || (lead_b && my_b >= T.cap_beliefs)) {
      T.counters[2] = 1;  // overflow: the host fails the plan loudly
      lead_a = lead_b = false;
    }
    const u64 word_a = ((u64)pass << 32) | (u64)(u32)my_a, word_b = ((u64)pass << 32) | (u64)(u32)my_b;
    Claim cl_a{0, false, 0}, cl_b{0, false, 0};
    {
      ClaimTry ta = claim_try_id(ha, T.hmask_a, key_a, word_a, lead_a);
      ClaimTry tb = claim_try_id(hb, T.hmask_b, key_b, word_b, lead_b);  // in flight together with ta
      if (lead_a) cl_a = claim_finish_id(ha, T.hmask_a, key_a, word_a, ta);
      if (lead_b) cl_b = claim_finish_id(hb, T.hmask_b, key_b, word_b, tb);
    }
    VP_PH(3);
    // deferred from the previous level: the overlay slot of the action this lane created there
    // (its atomic has had a whole level to return)
    if (pend_x >= 0) {
      T.a_slot[pend_x] = pend_k;
      if (!Exact && pend_k == kOverlay && pend_bel >= 0) pend_mat = pend_bel;  // dense row: after the levels
      pend_x = -1;
    }
    if (pend_mat >= 0 && pend_mat_prev >= 0) {  // a second one before the end: write the first now
      materialise_dense<PsiT>(T, W.stats, pend_mat_prev, load_rec<PsiT>(T, pend_mat_prev), init_row, pass);
      pend_mat_prev = -1;
    }
    if (pend_mat >= 0) {
      pend_mat_prev = pend_mat;
      pend_mat = -1;
    }
    // (belief, action, obs) keys: the child is known now -- resolve it and start loading its
    // record and LSE, so the action's bookkeeping below hides the load
    int c = 0;
    u32 cpass = 0;
    bool c_new = false, led_b = false;
    Rec<PsiT> rec_n{};
    double lse_n = lse_init;
    if (early) {
      if (lead_b) {
        const u64 w = wait_published(hb, cl_b.slot, cl_b.word);
        c = (int)(u32)w;
        cpass = (u32)(w >> 32);
      }
      c = __shfl_sync(FULL, c, leader_b);
      c_new = __shfl_sync(FULL, cpass, leader_b) == pass;
      led_b = __shfl_sync(FULL, (int)lead_b, leader_b) != 0;
      if constexpr (!Exact)
        if (ok && led_b && !c_new) {
          rec_n = load_rec<PsiT>(T, c);
          lse_n = T.b_lse[c];
        }
    }
    int x = 0;
    if (lead_a) {
      const u64 w = wait_published(ha, cl_a.slot, cl_a.word);  // (append kernels publish late)
      x = (int)(u32)w;
      if ((u32)(w >> 32) == pass) red_min(&T.a_ckey[x], creation_key(pass, l, rg));
    }
    if (cl_a.won) {
      // accumulators are zero (cleared at tree reset); the key is a min-reduction (above)
      T.a_parent_belief[x] = b;
      T.a_action[x] = a;
      pend_x = x;
      pend_bel = rec.dense_pass == 0 ? b : -1;
      if constexpr (!Exact) pend_k = atomicAdd(&T.b_nact[b], 1);  // consumed next level
      ++won_a;
    }
    x = __shfl_sync(FULL, x, leader_a);
    if (W.stats) {
      const u32 wn = __ballot_sync(FULL, cl_a.won);
      if (lane == 0 && wn) atomicAdd(&W.stats[5], (unsigned long long)__popc(wn));
    }
    // rewards and visits (tree.py:216-217); rows through x for the backup
    {
      const double sum = group_sum(rw, grp_a, ok);
      if (lead_a && ok) {
        const int cnt = __popc(grp_a);
        red_add(&T.a_reward[x], sum);
        red_add(&T.a_visits[x], cnt);
        red_add(&T.a_rows[x], cnt);
      }
    }
    const bool led_a = __shfl_sync(FULL, (int)lead_a, leader_a) != 0;  // (every lane shuffles)
    ok = ok && led_a;
    if (!early) {  // (action row, obs) keys: the belief claim needs x
      key_b = belief_key(T, b, a, x, o);
      grp_b = __match_any_sync(FULL, ok ? key_b : kEmptyKey);
      leader_b = __ffs(grp_b) - 1;
      lead_b = ok && lane == leader_b;
      if (lead_b && my_b >= T.cap_beliefs) {
        T.counters[2] = 1;
        lead_b = false;
      }
      if (lead_b) cl_b = claim_finish_id(hb, T.hmask_b, key_b, word_b, claim_try_id(hb, T.hmask_b, key_b, word_b, true));
    }
    VP_PH(4);
    grp = grp_b;
    lead = lead_b;
    {
      if (lead_b) {
        if (!early) {
          const u64 w = wait_published(hb, cl_b.slot, cl_b.word);
          c = (int)(u32)w;
          cpass = (u32)(w >> 32);
        }
        if (cpass == pass) red_min(&T.b_ckey[c], creation_key(pass, l, rg));
      }
      if (cl_b.won) {
        T.b_parent_action[c] = x;
        T.b_parent_obs[c] = o;
        T.b_parent_belief[c] = b;
        T.b_parent_act[c] = a;
        T.b_depth[c] = l + 1;
        T.b_lse[c] = lse_init;
        // fresh (PSI == init); an interior node's row is written by its creator next level
        T.b_flags[c] = interior_next ? 1u : 3u;
        ++won_b;
      }
      if (!early) {
        c = __shfl_sync(FULL, c, leader_b);
        c_new = __shfl_sync(FULL, cpass, leader_b) == pass;
      }
      made_interior = cl_b.won && interior_next;
      if (W.stats) {
        const u32 wn = __ballot_sync(FULL, cl_b.won);
        if (lane == 0 && wn) atomicAdd(&W.stats[6], (unsigned long long)__popc(wn));
      }
    }
    if (!early) led_b = __shfl_sync(FULL, (int)lead_b, leader_b) != 0;
    ok = ok && led_b;
    VP_PH(5);
    arrive(T, W, leaf_count, c, grp, lead && ok, !interior_next);
    if (active && W.trace_action) {
      const size_t t = (size_t)l * n + r;
      W.trace_action[t] = a;
      W.trace_obs[t] = o;
      W.trace_anode[t] = x;
      W.trace_belief[t] = c;
    }
    b = c;
    if constexpr (Exact) fl = c_new ? (interior_next ? 1u : 3u) : (ok ? T.b_flags[c] : 0u);
    if constexpr (!Exact) {
      if (c_new || !ok) {  // created this pass: the initial row
        rec = Rec<PsiT>{};
        lse = lse_init;
      } else if (early) {  // loaded during this level's bookkeeping
        rec = rec_n;
        lse = lse_n;
      } else {
        rec = load_rec<PsiT>(T, c);
        lse = T.b_lse[c];
      }
    }
  }

  if (pend_x >= 0) {
    T.a_slot[pend_x] = pend_k;
    if (!Exact && pend_k == kOverlay && pend_bel >= 0) pend_mat = pend_bel;
  }
  if constexpr (!Exact) {
    if (pend_mat_prev >= 0) materialise_dense<PsiT>(T, W.stats, pend_mat_prev, load_rec<PsiT>(T, pend_mat_prev), init_row, pass);
    if (pend_mat >= 0) materialise_dense<PsiT>(T, W.stats, pend_mat, load_rec<PsiT>(T, pend_mat), init_row, pass);
  }
  won_a = warp_sum(won_a);
  won_b = warp_sum(won_b);
  if (lane == 0) {
    if (won_a) red_add(&T.counters[VP_COUNTER_LIVE_A], won_a);
    if (won_b) red_add(&T.counters[VP_COUNTER_LIVE_B], won_b);
  }

  VP_PH(6);
  // ---- leaves: heuristic value (search.py:119), summed per leaf (backup.py:44-51)
  double h = 0.0;
  if (active) {
    h = !ok ? 0.0 : insert ? S.inject_leaf[r] : Model::heuristic(M, st);
    W.leaf_belief[r] = b;
    W.leaf_value[r] = h;
  }
  grp = __match_any_sync(FULL, ok ? (u32)b : 0xffffffffu);
  const double sum = group_sum(h, grp, ok);
  if (ok && lane == __ffs(grp) - 1) red_add(&T.b_value[b], sum);
  bulk_store_drain();
  VP_PH(7);
  VP_PH_FLUSH();
  if (W.stats && threadIdx.x == 0 && blockIdx.x == 0) {
    atomicAdd(&W.stats[3], 1ull);
    atomicAdd(&W.stats[4], (unsigned long long)n * (unsigned long long)(d - depth0));
  }
}

// ------------------------------------------------------------------ backup

// LSE of the rows held by the lanes in `rmask` (lane j's row is ready[j]);
// results land in out[j].  Rows are read from L2: their cells were written by
// other SMs inside this kernel.
template <class PsiT, bool Exact>
__device__ __forceinline__ void lse_ready(const vp_tree& T, int ready, u32 rmask, double* out) {
  const int A = T.action_count;
  const PsiT* psi = reinterpret_cast<const PsiT*>(T.psi);
  if constexpr (Exact) {
    if (ready >= 0) out[lane_id()] = lse_exact<true>(reinterpret_cast<const double*>(psi) + (size_t)ready * T.psi_stride,
                                                      A, T.eta);
  } else {
    // the fallback of the incremental LSE, fp64 arithmetic: the k rows are read in parallel,
    // each by a group of G = 32 / 2^ceil(log2 k) lanes (the completions that need it cluster
    // at the busy top levels, where a row-at-a-time loop put k full reads on the critical path)
    const int k = __popc(rmask);
    const int G = k <= 1 ? 32 : k <= 2 ? 16 : k <= 4 ? 8 : k <= 8 ? 4 : k <= 16 ? 2 : 1;
    const int lane = lane_id(), grp = lane / G, gl = lane % G;
    int owner = -1;  // the grp-th lane of rmask
    {
      u32 m = rmask;
      for (int i = 0; i < grp && m; ++i) m &= m - 1u;
      if (grp < k) owner = __ffs(m) - 1;
    }
    const int row = __shfl_sync(FULL, ready, owner >= 0 ? owner : 0);
    const PsiT* r = owner >= 0 ? psi + (size_t)row * T.psi_stride : nullptr;
    // one pass over the row, 8 loads in flight per lane, online max rescaling (the row lives
    // in L2: a load-then-use loop would pay one L2 round trip per element)
    double mx = -INFINITY, sm = 0.0;
    if (r) lse_online_f64<PsiT>(r, A, gl, G, T.eta, mx, sm);
    for (int o = G / 2; o > 0; o >>= 1) {
      const double m2 = __shfl_xor_sync(FULL, mx, o), s2 = __shfl_xor_sync(FULL, sm, o);
      const double mn = fmax(mx, m2);
      sm = (mx == -INFINITY ? 0.0 : sm * exp(mx - mn)) + (m2 == -INFINITY ? 0.0 : s2 * exp(m2 - mn));
      mx = mn;
    }
    if (owner >= 0 && gl == 0) out[owner] = mx / T.eta + log(sm) / T.eta;
  }
  __syncwarp();
}

// LSE of an overlay row (initial row + the record's realised cells) by one lane in fp64:
// the rare fallback of the incremental backup LSE.  The record is read from L2.
template <class PsiT>
__device__ __noinline__ double lse_overlay(const vp_tree& T, int b) {
  const Rec<PsiT> r = load_rec<PsiT, true>(T, b);
  const int A = T.action_count;
  const double eta = T.eta;
  auto val = [&](int a) -> double {
    double v = (double)(PsiT)T.init_prefs[a];
#pragma unroll
    for (int k = 0; k < kOverlay; ++k)
      if (r.act[k] == a + 1) v = (double)r.val[k];
    return v;
  };
  double m = -INFINITY;
  for (int a = 0; a < A; ++a) m = fmax(m, eta * val(a));
  double s = 0.0;
  for (int a = 0; a < A; ++a) s += exp(eta * val(a) - m);
  return m / eta + log(s) / eta;
}

// One warp = up to 32 distinct leaves; each lane climbs while it is the last
// arrival of the node above it.
template <class PsiT, bool Exact>
__device__ void backup_warp(const vp_tree& T, const vp_work& W, u32 pass, double gamma, int warp_index,
                            double* s_v, int rpw) {
  const int lane = lane_id();
  const int cnt = W.leaf_count[pass & 1u];
  const int i = lane < rpw ? warp_index * rpw + lane : INT_MAX;
  PsiT* psi = reinterpret_cast<PsiT*>(T.psi);
  const double eta = T.eta;
  int c = -1, rows = 0;
  double V = 0.0;
  u32 N = 0;
  if (i < cnt) {
    // leaf: V = mean heuristic, N = batch count (backup.py:44-51, 82-87)
    c = W.leaves[i];
    rows = T.b_rows[c];
    N = (u32)rows;
    V = T.b_value[c] / (double)rows;
    T.b_value[c] = 0.0;
    T.b_rows[c] = 0;
  }
  bool live = c >= 0;
  // the climb's pointers: parent action x, parent belief pb and the action label of c
  int x = -1, pb = -1, act = 0;
  if (live) {
    x = T.b_parent_action[c];
    pb = T.b_parent_belief[c];
    act = T.b_parent_act[c];
  }
  unsigned long long n_act = 0, n_bel = 0, n_psi = 0, n_cdf = 0, n_ovf = 0;
  VP_BK_INIT();
  VP_WAVE_DECL();
  if (lane == 0) VP_WAVE(pass, 63);
  while (__any_sync(FULL, live)) {
    VP_BK(0);
    int ready = -1, nx = -1, npb = -1, nact = 0;
#ifdef VP_PHASE_CLOCKS
    int bdel_pb = -1;
#endif
    int prow = -1;  // the PSI row of a completed belief's full-row fallback (-1: overlay row)
    u32 slotbit = 0, bmask = 0;  // overlay slot this lane's action changed / all changed slots
    Rec<PsiT> prec{};            // fast mode: the parent belief's overlay record
    double lse_pre = 0.0, bsum = 0.0;
    u32 bcnt = 0, btot = 0;
    bool fresh = false;
    if (live) {
      live = false;
      if (x >= 0) {
        // ONE round trip for everything a completing delivery needs -- the action's
        // statistics, the parent belief's LSE / rows, its PSI cell (parity mode) or overlay
        // record + the action's slot (fast mode) -- and the next level's pointers.  All of it
        // is stable until this lane completes the nodes.
        const int tot = T.a_rows[x], vis = T.a_visits[x];
        const double rew = T.a_reward[x];
        lse_pre = T.b_lse[pb];
        btot = (u32)T.b_rows[pb];
        PsiT* cell = nullptr;
        double old_v = 0.0, init_v = 0.0;
        int slot = 0;
        if constexpr (Exact) {
          cell = psi + (size_t)pb * T.psi_stride + act;
          old_v = (double)__ldcg(cell);
        } else {
          prec = load_rec<PsiT>(T, pb);  // slots untouched this pass are stable in this kernel
          slot = T.a_slot[x];
          init_v = T.init_prefs[act];
        }
        nx = T.b_parent_action[pb];
        npb = T.b_parent_belief[pb];
        nact = T.b_parent_act[pb];
        // child mean of the action (backup.py:64-68): sum V*N, sum N
        Acc aa;
        if (acc_deliver(T.a_acc, x, V * (double)N, (u32)rows, N, (u32)tot, aa)) {
          // last child: Q (backup.py:96-104) and PSI[b, a] += Q - LSE_pre(b) (:106-108)
          ++n_act;
          T.a_rows[x] = 0;
          // fp32 storage: Q enters a cell rounded to fp32 anyway -- fp32 reciprocals (MUFU) suffice
          const double q = sizeof(PsiT) == 4 && !Exact
                               ? (double)__fdividef((float)rew, (float)vis) +
                                     (double)__fdividef((float)(gamma * aa.sum), (float)aa.cnt)
                               : rew / (double)vis + (gamma * aa.sum) / (double)aa.cnt;
          double term = 0.0;
          if constexpr (Exact) {
            *cell = (PsiT)(old_v + (q - lse_pre));
            __threadfence();  // the full-row LSE of pb reads this cell from another SM
          } else {
            // LSE_pre is the row's LSE, so LSE_post follows from the changed cells:
            // sum_a exp(eta (psi_a - LSE_pre)) = 1 + sum_changed (new - old)
            fresh = true;
            const bool dense = prec.dense_pass != 0;
            if (dense) {
              prow = (int)prec.dense_row;
              cell = psi + (size_t)prow * T.psi_stride + act;
              old_v = (double)__ldcg(cell);
            } else if (slot < kOverlay) {
              old_v = prec.act[slot] ? (double)prec.val[slot] : (double)(PsiT)init_v;
            } else {
              T.counters[2] = 1;  // a child beyond the overlay without a dense row: fail loudly
            }
            const PsiT new_v = (PsiT)(old_v + (q - lse_pre));
            if (dense) {
              term = exp(eta * ((double)new_v - lse_pre)) - exp(eta * (old_v - lse_pre));
              *cell = new_v;  // published to the completer by the ordered delivery below
            } else if (slot < kOverlay) {
              // overlay row: deliver the new cell's log-mass eta psi and flag its slot; the
              // completing lane adds the unchanged cells (untouched slots + unrealised initial
              // cells) in log space, so nothing cancels, overflows or underflows
              term = eta * (double)new_v;
              slotbit = kSlotBit << slot;
              Rec<PsiT>* g = rec_ptr<PsiT>(T, pb);
              g->val[slot] = new_v;
              g->act[slot] = (unsigned short)(act + 1);
              if (!T.init_uniform) __threadfence();  // the general LSE reads every cell
            }
          }
          // N(b) = lifetime visits of the valued actions (backup.py:110-114)
#ifdef VP_PHASE_CLOCKS
          if ((u32)tot != btot) bdel_pb = pb;
#endif
          Acc ba;
          const bool done = slotbit ? acc_deliver_log(T.b_acc, pb, term, (u32)tot | slotbit, (u32)vis, btot, ba)
                            : prow >= 0 ? acc_deliver<true>(T.b_acc, pb, term, (u32)tot, (u32)vis, btot, ba)
                                        : acc_deliver(T.b_acc, pb, term, (u32)tot, (u32)vis, btot, ba);
          if (done) {
            ready = pb;
            bsum = ba.sum;
            bcnt = ba.cnt;
            bmask = ba.rows >> 24;
          }
        }
      }
    }
#ifdef VP_PHASE_CLOCKS
    {  // how many multi-delivery belief deliveries of this iteration share their belief in the warp
      const u32 g_ = __match_any_sync(FULL, bdel_pb);
      const bool d_ = bdel_pb >= 0, l_ = d_ && lane == __ffs(g_) - 1;
      const u32 nd_ = __popc(__ballot_sync(FULL, d_)), ng_ = __popc(__ballot_sync(FULL, l_));
      if (lane == 0 && nd_) {
        atomicAdd(&g_phase_cycles[20], (unsigned long long)nd_);
        atomicAdd(&g_phase_cycles[21], (unsigned long long)ng_);
      }
    }
#endif
    VP_BK(1);
    if (__any_sync(FULL, ready >= 0)) {
      // last action of a belief: V = LSE_post (backup.py:109), cached as the next LSE_pre.
      // Fast mode uses the incremental sum; parity mode (and tiny / overflowing incremental
      // sums) read the row in full -- the warp for PSI rows, the lane for an overlay row.
      bool full = ready >= 0;
      bool ofull = false;
      if constexpr (!Exact) {
        // overlay row (uniform initial row): eta LSE = log sum_a exp(eta psi_a) = the changed
        // cells (delivered, log space) (+) the slots untouched this pass (stable in this lane's
        // record) (+) the unrealised initial cells, (|A| - filled) exp(eta init): one max shift,
        // then only the exponentials some lane of the warp needs (the max term is exactly 1 --
        // typically one exponential and one log per belief)
        const bool ovl = ready >= 0 && fresh && prow < 0 && T.init_uniform;
        double lk[kOverlay];
        double m = ovl ? bsum : 0.0;
        int filled = __popc(bmask);
#pragma unroll
        for (int k = 0; k < kOverlay; ++k) {
          const bool keep = ovl && !((bmask >> k) & 1u) && prec.act[k];
          lk[k] = keep ? eta * (double)prec.val[k] : -INFINITY;
          m = fmax(m, lk[k]);
          filled += keep;
        }
        const double li = eta * (double)(PsiT)T.init_prefs[0];
        const int rest = T.action_count - filled;
        if (ovl && rest > 0) m = fmax(m, li);
        // fp32 storage: the terms lie in (0, 1] and the sum in [1, |A| + 4], so fp32 exp / log
        // (MUFU) give the LSE to ~1e-7 of its scale -- inside the 1e-5 scale-aware contract
        // and at the accuracy of the stored cells themselves; fp64 storage keeps fp64 math
        constexpr bool kF32 = sizeof(PsiT) == 4;
        auto term = [&](bool use, double x) -> double {  // exp(x - m) for the lanes that use it
          const bool need = use && x != m;
          double t = use ? 1.0 : 0.0;
          if (__any_sync(FULL, need)) {
            const double e = kF32 ? (double)__expf((float)(x - m)) : exp(x - m);
            if (need) t = e;
          }
          return t;
        };
        double sum = term(ovl, bsum) + (double)rest * term(ovl && rest > 0, li);
#pragma unroll
        for (int k = 0; k < kOverlay; ++k) sum += term(lk[k] > -INFINITY, lk[k]);
        if (ovl) {
          V = (m + (kF32 ? (double)__logf((float)sum) : log(sum))) / eta;
          full = false;
        } else if (fresh && prow >= 0) {
          // dense row: 1 + sum_changed (new - old) relative to its exact (fp64-maintained) LSE.
          // Each term carries the rounding of eta (psi - LSE) (~|A| ulp(|psi|) in all), so the
          // sum's relative error is ~|A| ulp(|psi|) / sum: trusted down to 1e-3 for fp32 storage
          // (<= 1e-8 relative, far inside its 1e-5 contract) and 0.9 for fp64 (1e-10 contract);
          // below that the warp reads the row
          constexpr double kTrust = sizeof(PsiT) == 4 ? 1e-3 : 0.9;
          const double sum = 1.0 + bsum;
          if (sum > kTrust && sum < 1e300) {
            V = lse_pre + log(sum) / eta;
            full = false;
          }
        }
        ofull = full && prow < 0;
        if (ofull) {  // overlay row of a non-uniform initial row: every writer fenced
          __threadfence();
          V = lse_overlay<PsiT>(T, ready);
        }
      }
      const u32 fmask = __ballot_sync(FULL, full && !ofull);
      if (fmask) {
        __threadfence();
        lse_ready<PsiT, Exact>(T, full && !ofull ? (Exact ? ready : prow) : -1, fmask, s_v);
      }
      if (ready >= 0) {
        ++n_bel;
        if (full) {
          if (!ofull) V = s_v[lane];
          ++n_psi;
          n_ovf += ofull;
        }
        if constexpr (!Exact)
          if (prow >= 0) {  // a changed dense row: the CDF kernel after this one rebuilds its CDF
            DenseMeta* dm = reinterpret_cast<DenseMeta*>(T.dense_meta) + prow;
            dm->lse = V;
            dm->pass = pass;
            ++n_cdf;
          }
        VP_WAVE(pass, min(T.b_depth[ready], 62));
        T.b_lse[ready] = V;
        T.b_flags[ready] = 0u;
        T.b_rows[ready] = 0;
        N = bcnt;
        rows = (int)btot;
        c = ready;
        x = nx;
        pb = npb;
        act = nact;
        live = true;
      }
    }
  }
  VP_BK(2);
  VP_WAVE_FLUSH();
  if (W.stats) {
    n_act = warp_sum(n_act);
    n_bel = warp_sum(n_bel);
    n_psi = warp_sum(n_psi);
    n_cdf = warp_sum(n_cdf);
    n_ovf = warp_sum(n_ovf);
    if (lane == 0) {
      if (n_bel) atomicAdd(&W.stats[0], n_bel);
      if (n_psi) atomicAdd(&W.stats[8], n_psi);
      if (n_act) atomicAdd(&W.stats[1], n_act);
      if (n_cdf) atomicAdd(&W.stats[11], n_cdf);
      if (n_ovf) atomicAdd(&W.stats[12], n_ovf);
      if (i < cnt) atomicAdd(&W.stats[7], (unsigned long long)min(rpw, cnt - warp_index * rpw));
    }
  }
}

// The dense rows a backup changed get their softmax CDF rebuilt for the next pass's draws, one
// warp per row over the whole GPU (off the backup's climb; the kernel boundary makes every new
// cell visible).
template <class PsiT>
__device__ void cdf_rows_warp(const vp_tree& T, u32 pass) {
  const int nd = min(T.counters[VP_COUNTER_DENSE], T.cap_dense);
  const int warps = gridDim.x * (blockDim.x >> 5);
  const PsiT* psi = reinterpret_cast<const PsiT*>(T.psi);
  PsiT* cdf = reinterpret_cast<PsiT*>(T.psi_cdf);
  const DenseMeta* meta = reinterpret_cast<const DenseMeta*>(T.dense_meta);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nd; r += warps) {
    const DenseMeta m = meta[r];
    if (m.pass == pass)
      build_cdf_row<PsiT, false>(psi + (size_t)r * T.psi_stride, cdf + (size_t)r * T.psi_stride, T.action_count,
                                 T.eta, m.lse);
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
