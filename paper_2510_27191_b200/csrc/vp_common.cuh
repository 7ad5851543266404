// vp_common.cuh -- device building blocks of the PORPP planning step (sm_100a).
//
//  * counter-hash RNG, bit-identical to the reference RowRng
//    (/root/reference/pkg/src/vecpomdp/rng.py:26-89);
//  * open-addressing hash index claimed with one 128-bit CAS per probe
//    (replaces tree.py:44-68 sorted-cache matching);
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

// ---------------------------------------------------------------- Philox fast mode
//
// vp_model.rng_kind = VP_RNG_PHILOX replaces the per-row SplitMix64 hash by
// Philox4x32-10 (Salmon et al., SC'11; the constants of curand_philox4x32_x.h;
// pinned to the Random123 known-answer vectors, tests/test_gpu_philox.py).  The
// stream keys (derive / fold: warp-uniform) are unchanged; a row's draw j of
// the stream `key` is the block
//   Philox4x32-10(counter = {lo(row), hi(row), lo(j), tag}, key = {lo(key), hi(key)})
// with tag 0 for uniforms (j = 0: the single draw, j >= 1: the j-th of k) and
// tag 1 for normals.  A uniform takes the top 53 bits of {x, y}.  Normals come
// in Box-Muller pairs: block b = (j + 1) / 2 gives u1 = bits{x, y} + 1 ulp,
// u2 = bits{z, w}, R = sqrt(-2 log u1); normal j is R cos(2 pi u2) for odd j (and
// j = 0), R sin(2 pi u2) for even j -- one block, one log and one sqrt per pair.
// Not the reference's streams: trees differ from the reference's, their
// statistics do not (oracle/rng.py: philox4x32_10, PhiloxRowRng).
constexpr u32 kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
constexpr u32 kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const u32 lo0 = kPhiloxM0 * c.x, hi0 = __umulhi(kPhiloxM0, c.x);
    const u32 lo1 = kPhiloxM1 * c.z, hi1 = __umulhi(kPhiloxM1, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += kPhiloxW0;
    k.y += kPhiloxW1;
  }
  return c;
}
__device__ __forceinline__ uint4 philox_block(u64 key, u64 row, u64 j, u32 tag) {
  return philox4x32_10(make_uint4((u32)row, (u32)(row >> 32), (u32)j, tag), make_uint2((u32)key, (u32)(key >> 32)));
}
__device__ __forceinline__ double philox_unit(u64 key, u64 row, u64 j) {
  const uint4 b = philox_block(key, row, j, 0u);
  return unit53(((u64)b.x << 32) | b.y);
}
// the pair of block b: (R cos, R sin)
__device__ __forceinline__ double2 philox_normal_pair(u64 key, u64 row, u64 b) {
  const uint4 h = philox_block(key, row, b, 1u);
  const double u1 = ((double)((((u64)h.x << 32) | h.y) >> 11) + 1.0) * kInv53;
  const double u2 = (double)((((u64)h.z << 32) | h.w) >> 11) * kInv53;
  const double r = sqrt(-2.0 * log(u1));
  return make_double2(r * cos(kTwoPi * u2), r * sin(kTwoPi * u2));
}
__device__ __forceinline__ double philox_normal(u64 key, u64 row, u64 j) {
  const double2 z = philox_normal_pair(key, row, (j + 1) >> 1);
  return (j == 0 || (j & 1)) ? z.x : z.y;
}

// Stream-kind dispatch (rk = vp_model.rng_kind: kernel-parameter uniform, no divergence).
__device__ __forceinline__ double uniform1(u64 key, u64 row, int rk) {
  return rk ? philox_unit(key, row, 0) : uniform1(key, row);
}
__device__ __forceinline__ double uniform_j(u64 key, u64 row, u64 j, int rk) {
  return rk ? philox_unit(key, row, j) : uniform_j(key, row, j);
}
__device__ __forceinline__ double normal_j(u64 key, u64 row, u64 j, int rk) {
  return rk ? philox_normal(key, row, j) : normal_j(key, row, j);
}
// A row's stream handle for many draws: SplitMix64 precomputes the row base
// (rng.py:69); Philox keeps the key and takes the row per draw.
__device__ __forceinline__ u64 stream_base(u64 key, u64 row, int rk) { return rk ? key : row_base(key, row); }
__device__ __forceinline__ double stream_uniform(u64 base, u64 row, u64 j, int rk) {
  return rk ? philox_unit(base, row, j) : unit53(mix64(base + j * kMixB));
}

// ---------------------------------------------------------------- hashing

// 16-byte slot of an open-addressing index.  Empty slots are all-ones (one
// memset).  A claim is ONE 128-bit CAS on an empty slot: the search inserts
// {key, pass | id} at once (its ids are static, known before the claim); the
// host-level append kernels insert {key, unpublished}, number the node and
// publish {id, pass} with a 64-bit store.  A loser gets the whole slot back
// from the failed CAS, so a hit costs one L2 round trip.
struct __align__(16) Slot {
  u64 key;
  u32 id;    // node id, kUnpublished while the winner is still numbering it
  u32 pass;  // search pass that created the node (0 after a rehash)
};
constexpr u64 kEmptyKey = ~0ull;
constexpr u32 kUnpublished = 0xffffffffu;

__device__ __forceinline__ u64 slot_hash(u64 key) { return mix64(key ^ 0x5851F42D4C957F2Dull); }

__device__ __forceinline__ u32 ld_volatile_u32(const u32* p) { return *(volatile const u32*)p; }
// gpu-scope relaxed loads read L2 (never a stale L1 line written by another SM)
__device__ __forceinline__ u32 ld_relaxed_u32(const u32* p) {
  u32 v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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
__device__ __forceinline__ u64 ld_acquire_u64(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// fire-and-forget reductions (REDG): nothing waits for them inside a kernel
__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void red_add(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_min(uint64_t* p, u64 v) {
  asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// acq_rel add: releases this thread's earlier writes (REDs included) and
// acquires everything released by earlier adders of the same counter.
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void cas128(void* p, u64 cmp_lo, u64 cmp_hi, u64 new_lo, u64 new_hi, u64& old_lo,
                                       u64& old_hi) {
  asm volatile(
      "{\n .reg .b128 c, n, d;\n mov.b128 c, {%2, %3};\n mov.b128 n, {%4, %5};\n"
      " atom.relaxed.gpu.global.cas.b128 d, [%6], c, n;\n mov.b128 {%0, %1}, d;\n}\n"
      : "=l"(old_lo), "=l"(old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(new_lo), "l"(new_hi), "l"(p)
      : "memory");
}

// Result of a claim: the slot, whether this thread created the key, and --
// for a hit -- the published {id, pass} word (id == kUnpublished: the
// creator has not numbered it yet; spin with wait_published).
struct Claim {
  u32 slot;
  bool won;
  u64 word;  // id | pass << 32
};

__device__ __forceinline__ Claim claim_key(Slot* tab, u64 mask, u64 key) {
  u64 h = slot_hash(key) & mask;
  while (true) {
    u64 old_key, old_word;
    cas128(&tab[h], kEmptyKey, ~0ull, key, ~0ull, old_key, old_word);
    if (old_key == kEmptyKey) return Claim{(u32)h, true, ~0ull};
    if (old_key == key) return Claim{(u32)h, false, old_word};
    h = (h + 1) & mask;
  }
}

// Publication needs no release: everything other rows touch inside the
// search kernel is either an accumulator (zero before the pass, updated with
// L2 reductions) or derived from the slot word itself (the creating pass);
// the columns the creator writes are read only by later kernels.
__device__ __forceinline__ void publish(Slot* tab, u32 slot, u32 id, u32 pass) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(&tab[slot].id), "l"(((u64)pass << 32) | id) : "memory");
}

__device__ __forceinline__ u64 wait_published(const Slot* tab, u32 slot, u64 word) {
  const u64* p = reinterpret_cast<const u64*>(&tab[slot].id);
  while ((u32)word == kUnpublished) word = ld_relaxed_u64(p);
  return word;
}

// Plain insert of a known (key, id) pair; used by rehash (pass 0 = "old").
__device__ __forceinline__ void put_final(Slot* tab, u64 mask, u64 key, u32 id) {
  u64 h = slot_hash(key) & mask;
  while (true) {
    const u64 prev = atomicCAS(&tab[h].key, kEmptyKey, key);
    if (prev == kEmptyKey || prev == key) {
      tab[h].id = id;
      tab[h].pass = 0;
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
