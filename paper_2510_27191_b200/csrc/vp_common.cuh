// vp_common.cuh -- device building blocks of the PORPP planning step (sm_100a).
//
//  * counter-hash RNG, bit-identical to the reference RowRng
//    (/root/reference/pkg/src/vecpomdp/rng.py:26-89);
//  * open-addressing hash index with deterministic first-occurrence ids
//    (replaces tree.py:44-68 sorted-cache matching);
//  * decoupled look-back tile scan used to number new nodes in batch order;
//  * numpy-order pairwise summation (for the fp64 parity mode).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/vpb200.h"

namespace vp {

typedef unsigned long long u64;
typedef uint32_t u32;

constexpr u64 kPhi = 0x9E3779B97F4A7C15ull;
constexpr u64 kMixA = 0xBF58476D1CE4E5B9ull;
constexpr u64 kMixB = 0x94D049BB133111EBull;
constexpr double kInv53 = 1.0 / 9007199254740992.0;  // 2^-53
constexpr double kTwoPi = 6.283185307179586;         // fl(2 * pi), rng.py:23
constexpr u32 FULL = 0xffffffffu;

// ---------------------------------------------------------------- RNG

__host__ __device__ __forceinline__ u64 mix64(u64 x) {  // rng.py:26-31
  x = (x ^ (x >> 30)) * kMixA;
  x = (x ^ (x >> 27)) * kMixB;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ u64 fold(u64 key, u64 word) {  // rng.py:34-36
  return mix64(key + kPhi * (word + 1));
}
__device__ __forceinline__ u64 row_base(u64 key, u64 row) {  // rng.py:69
  return mix64(key + kPhi * (row + 2));
}
__device__ __forceinline__ double unit53(u64 h) { return (double)(h >> 11) * kInv53; }
// single draw (k = None): rng.py:70-71
__device__ __forceinline__ double uniform1(u64 key, u64 row) { return unit53(mix64(row_base(key, row) + kMixA)); }
// j-th of k draws, j = 1..k: rng.py:72-73
__device__ __forceinline__ double uniform_j(u64 key, u64 row, u64 j) {
  return unit53(mix64(row_base(key, row) + j * kMixB));
}
// Box-Muller normal; j = 0 means the single-draw form (rng.py:81-89)
__device__ __forceinline__ double normal_j(u64 key, u64 row, u64 j) {
  const u64 k1 = fold(key, 101), k2 = fold(key, 211);
  const u64 b1 = row_base(k1, row), b2 = row_base(k2, row);
  const u64 h1 = mix64(b1 + (j ? j * kMixB : kMixA));
  const u64 h2 = mix64(b2 + (j ? j * kMixB : kMixA));
  const double u1 = ((double)(h1 >> 11) + 1.0) * kInv53;
  const double u2 = (double)(h2 >> 11) * kInv53;
  return sqrt(-2.0 * log(u1)) * cos(kTwoPi * u2);
}

// ---------------------------------------------------------------- hashing

struct __align__(16) Slot {
  u64 key;
  u32 id;   // final node id, or kPending|min_row while being claimed this level
  u32 pad;
};
constexpr u64 kEmptyKey = ~0ull;
constexpr u32 kEmptyId = 0xffffffffu;
constexpr u32 kPending = 0x80000000u;
constexpr u32 kExistBit = 0x80000000u;  // in per-row slot words

__device__ __forceinline__ u64 slot_hash(u64 key) { return mix64(key ^ 0x5851F42D4C957F2Dull); }

__device__ __forceinline__ u64 ld_volatile_u64(const u64* p) { return *(volatile const u64*)p; }
__device__ __forceinline__ u32 ld_volatile_u32(const u32* p) { return *(volatile const u32*)p; }
// gpu-scope relaxed loads read L2 without invalidating L1 (an acquire would
// emit CCTL.IVALL and throw away every warp's L1 lines on the SM).
__device__ __forceinline__ u32 ld_relaxed_u32(const u32* p) {
  u32 v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 ld_relaxed_u64(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u32 ld_relaxed_u8(const uint8_t* p) {
  unsigned short v;
  asm volatile("ld.relaxed.gpu.global.u8 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
  return (u32)v;
}
__device__ __forceinline__ u32 ld_acquire_u32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(u32* p, u32 v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire_u64(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Find or claim `key`.  Returns the slot index; sets `existing` when the key
// already carried a final id from an earlier phase.  New keys record the
// minimum claiming row (first occurrence) via atomicMin on the id word; the
// returned old id tells hits (< kPending) from claims, so a probe costs two
// L2 atomics (CAS on the key, min on the id) and no plain loads.
__device__ __forceinline__ u32 probe_claim(Slot* tab, u64 mask, u64 key, u32 row, bool& existing, u32& id) {
  u64 h = slot_hash(key) & mask;
  while (true) {
    const u64 prev = atomicCAS(&tab[h].key, kEmptyKey, key);
    if (prev == kEmptyKey || prev == key) {
      const u32 old = atomicMin(&tab[h].id, kPending | row);
      existing = old < kPending;
      id = existing ? old : kEmptyId;
      return (u32)h;
    }
    h = (h + 1) & mask;
  }
}

// Plain insert of a known (key, id) pair; used by rehash.
__device__ __forceinline__ void put_final(Slot* tab, u64 mask, u64 key, u32 id) {
  u64 h = slot_hash(key) & mask;
  while (true) {
    const u64 prev = atomicCAS(&tab[h].key, kEmptyKey, key);
    if (prev == kEmptyKey || prev == key) {
      tab[h].id = id;
      return;
    }
    h = (h + 1) & mask;
  }
}

// ---------------------------------------------------------------- warp helpers

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(FULL, v, o);
    v = w > v ? w : v;
  }
  return v;
}
template <class T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T w = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += w;
  }
  return v;
}

// ---------------------------------------------------------------- tile scan

// Decoupled look-back: returns the exclusive prefix of `agg` over tiles in
// ticket order.  Status word: epoch(32) | flag(2) | value(30).
constexpr u64 kFlagAgg = 1, kFlagInc = 2;
__device__ __forceinline__ u64 pack_status(u32 epoch, u64 flag, u32 v) {
  return ((u64)epoch << 32) | (flag << 30) | (u64)(v & 0x3fffffffu);
}

__device__ __forceinline__ u32 tile_lookback(u64* status, int tile, u32 agg, u32 epoch) {
  // called by one thread
  if (tile == 0) {
    st_release_u64(&status[0], pack_status(epoch, kFlagInc, agg));
    return 0;
  }
  st_release_u64(&status[tile], pack_status(epoch, kFlagAgg, agg));
  u32 excl = 0;
  int j = tile - 1;
  while (true) {
    const u64 s = ld_acquire_u64(&status[j]);
    if ((u32)(s >> 32) != epoch) continue;  // predecessor not published yet
    excl += (u32)(s & 0x3fffffffu);
    if (((s >> 30) & 3) == kFlagInc) break;
    --j;
  }
  st_release_u64(&status[tile], pack_status(epoch, kFlagInc, excl + agg));
  return excl;
}

// Warp-parallel variant (called by all 32 lanes of one warp): each round
// inspects 32 predecessors at once, so a tile waits ~tiles/32 L2 round trips
// instead of one per predecessor.
__device__ __forceinline__ u32 tile_lookback_warp(u64* status, int tile, u32 agg, u32 epoch) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) st_release_u64(&status[tile], pack_status(epoch, tile == 0 ? kFlagInc : kFlagAgg, agg));
  if (tile == 0) return 0;
  u32 excl = 0;
  int base = tile - 1;
  while (true) {
    const int j = base - lane;
    const u64 s = j >= 0 ? ld_relaxed_u64(&status[j]) : pack_status(epoch, kFlagInc, 0);
    const bool valid = (u32)(s >> 32) == epoch;
    const u32 inc = __ballot_sync(0xffffffffu, valid && ((s >> 30) & 3) == kFlagInc);
    const u32 bad = __ballot_sync(0xffffffffu, !valid);
    const int limit = inc ? __ffs(inc) - 1 : 31;
    const u32 upto = limit == 31 ? 0xffffffffu : ((2u << limit) - 1u);
    if (bad & upto) continue;  // a needed predecessor has not published yet
    u32 v = lane <= limit ? (u32)(s & 0x3fffffffu) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
    base -= 32;
  }
  if (lane == 0) st_release_u64(&status[tile], pack_status(epoch, kFlagInc, excl + agg));
  return excl;
}

// ---------------------------------------------------------------- numpy-order sums

// numpy pairwise_sum for float64 (8 accumulators, 128-element blocks,
// recursive halving rounded to a multiple of 8), over f(lo..lo+n).
template <class F>
__device__ __forceinline__ double pairwise_leaf(const F& f, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += f(lo + i);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += f(lo + i + j);
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += f(lo + i);
  return res;
}

// The recursion of numpy's pairwise_sum, evaluated with an explicit stack
// (post-order: left half, right half, add) so the frame size is static.
template <class F>
__device__ double pairwise_sum(const F& f, int lo, int n) {
  if (n <= 128) return pairwise_leaf(f, lo, n);
  int s_lo[24], s_n[24], s_state[24];
  double s_left[24];
  int sp = 0;
  s_lo[0] = lo;
  s_n[0] = n;
  s_state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    const int cl = s_lo[sp], cn = s_n[sp];
    if (cn <= 128) {
      ret = pairwise_leaf(f, cl, cn);
      --sp;
      continue;
    }
    int n2 = cn / 2;
    n2 -= n2 % 8;
    if (s_state[sp] == 0) {
      s_state[sp] = 1;
      ++sp;
      s_lo[sp] = cl;
      s_n[sp] = n2;
      s_state[sp] = 0;
    } else if (s_state[sp] == 1) {
      s_left[sp] = ret;
      s_state[sp] = 2;
      ++sp;
      s_lo[sp] = cl + n2;
      s_n[sp] = cn - n2;
      s_state[sp] = 0;
    } else {
      ret = s_left[sp] + ret;
      --sp;
    }
  }
  return ret;
}

}  // namespace vp
