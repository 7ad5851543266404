// vp_models.cuh -- device generative models G(s, a) -> (s', o, r) and leaf
// heuristics.  Each model replays its host definition operation for
// operation so that integer outputs are bit-identical:
//   MARS      /root/reference/pkg/src/vecpomdp/envs/mars.py:146-180, 223-243
//   TABULAR   /root/reference/pkg/src/vecpomdp/envs/tabular.py:106-130
//   SYNTHETIC oracle/envs.py SyntheticModel   (new; integer hash dynamics)
//   LIGHTDARK oracle/envs.py LightDarkModel   (new; continuous observations)
//   NAVIGATION /root/reference/pkg/src/vecpomdp/envs/navigation.py:146-251
// The per-row model stream is `mkey` = level_rng.derive(1) (search.py:113-115)
// and the logical row id is the global simulation index.
#pragma once

#include "vp_common.cuh"

namespace vp {

// ------------------------------------------------------------------ MARS
// 16-byte packed record: agent columns/rows (x == n means departed), rock
// quality bits (bit i set while rock i is good), terminal flag.
struct __align__(16) MarsState {
  uint8_t x0, y0, x1, y1;
  uint32_t term;
  u64 rocks;
};

struct MarsModel {
  typedef MarsState State;
  static __device__ __forceinline__ void step(const vp_model& M, State& s, int a, u64 mkey, u64 row,
                                              u32& obs, double& rew, int rkind) {
    const int n = M.mars_n, P = M.mars_ops;
    const int op[2] = {a / P, a % P};
    const State in = s;
    const bool gone[2] = {in.x0 == n, in.x1 == n};
    int x[2] = {in.x0, in.x1}, y[2] = {in.y0, in.y1};
    u64 rocks = in.rocks;
    double part[4] = {0.0, 0.0, 0.0, 0.0};
    // moves N/E/S/W for both agents (mars.py:95-111, 154-155)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!gone[k] && op[k] < 4) {
        const int dx = (op[k] == 1) - (op[k] == 3);
        const int dy = (op[k] == 2) - (op[k] == 0);
        const int tx = x[k] + dx, ty = y[k] + dy;
        const bool departs = tx == n;
        const bool inside = tx >= 0 && tx < n && ty >= 0 && ty < n;
        if (departs || inside) {
          x[k] = tx;
          if (!departs) y[k] = ty;
        }
        if (departs) part[k] = 10.0;
      }
    }
    // samples, agent 0 first (mars.py:113-127, 156-157)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!gone[k] && op[k] == 4) {
        part[2 + k] = -10.0;
        const int rk = M.mars_rock_at[x[k] * n + y[k]];
        if (rk >= 0 && ((rocks >> rk) & 1ull)) {
          part[2 + k] = 10.0;
          rocks &= ~(1ull << rk);
        }
      }
    }
    // sensor readings from post-sample rocks (mars.py:129-144, 158-165)
    int reading[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double u = uniform1(fold(mkey, (u64)k), row, rkind);
      reading[k] = 2;  // NULL
      if (!gone[k] && op[k] >= 5) {
        const int rk = op[k] - 5;
        const int adx = abs(x[k] - M.mars_rock_x[rk]), ady = abs(y[k] - M.mars_rock_y[rk]);
        const double acc = M.mars_acc[adx * (n + 1) + ady];  // 0.5 (1 + 2^(-d / half_eff))
        const bool correct = u < acc;
        const bool truth = (rocks >> rk) & 1ull;
        reading[k] = (truth == correct) ? 0 : 1;
      }
    }
    obs = (u32)(reading[0] * 3 + reading[1]);
    rew = (((0.0 + part[0]) + part[1]) + part[2]) + part[3];
    const bool term = in.term || (x[0] == n && x[1] == n);
    if (term) obs = (u32)M.obs_arity;
    if (in.term) {
      rew = 0.0;
      return;  // absorbing: state unchanged (mars.py:174-179)
    }
    s.x0 = (uint8_t)x[0]; s.y0 = (uint8_t)y[0];
    s.x1 = (uint8_t)x[1]; s.y1 = (uint8_t)y[1];
    s.rocks = rocks;
    s.term = term ? 1u : 0u;
  }

  // log P(obs | s', a) for the SIR reweighting (mars.py:182-221)
  static __device__ __forceinline__ double obs_loglik(const vp_model& M, const State& s, int a, u32 obs) {
    if (obs == (u32)M.obs_arity) return s.term ? 0.0 : -INFINITY;
    if (s.term) return -INFINITY;
    const int n = M.mars_n, P = M.mars_ops;
    const int ops[2] = {a / P, a % P};
    const int want[2] = {(int)obs / 3, (int)obs % 3};  // GOOD 0, BAD 1, NULL 2
    const int xs[2] = {s.x0, s.x1}, ys[2] = {s.y0, s.y1};
    double logp = 0.0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      double p;
      if (ops[k] >= 5) {
        const int rk = ops[k] - 5;
        const double acc = M.mars_acc[abs(xs[k] - M.mars_rock_x[rk]) * (n + 1) + abs(ys[k] - M.mars_rock_y[rk])];
        const bool good = (s.rocks >> rk) & 1ull;
        p = want[k] == 0 ? (good ? acc : 1.0 - acc) : want[k] == 1 ? (good ? 1.0 - acc : acc) : 0.0;
        if (xs[k] == n) p = want[k] == 2 ? 1.0 : 0.0;
      } else {
        p = want[k] == 2 ? 1.0 : 0.0;
      }
      logp += log(p);
    }
    return logp;
  }

  static __device__ __forceinline__ double heuristic(const vp_model& M, const State& s) {
    // mars.py:223-243
    if (s.term) return 0.0;
    const int n = M.mars_n;
    const int xs[2] = {s.x0, s.x1}, ys[2] = {s.y0, s.y1};
    const bool act[2] = {xs[0] < n, xs[1] < n};
    double h = 0.0;
    h += act[0] ? 10.0 * M.mars_gpow[n - xs[0] - 1] : 0.0;
    h += act[1] ? 10.0 * M.mars_gpow[n - xs[1] - 1] : 0.0;
    if (!(act[0] || act[1])) return h;
    auto term_i = [&](int i) -> double {
      int best = 0x3fffffff;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (!act[k]) continue;
        const int dd = abs(xs[k] - M.mars_rock_x[i]) + abs(ys[k] - M.mars_rock_y[i]);
        best = dd < best ? dd : best;
      }
      const double good = ((s.rocks >> i) & 1ull) ? 10.0 : 0.0;
      return good * M.mars_gpow[best];
    };
    h += pairwise_leaf(term_i, 0, M.mars_m);  // numpy pairwise sum; m <= 64 < 128: one leaf block
    return h;
  }
};

// ------------------------------------------------------------------ TABULAR
struct __align__(8) TabularState {
  int32_t idx;
  int32_t term;
};

struct TabularModel {
  typedef TabularState State;
  static __device__ __forceinline__ void step(const vp_model& M, State& s, int a, u64 mkey, u64 row,
                                              u32& obs, double& rew, int rkind) {
    const int S = M.tab_states, O = M.tab_obs;
    const int cur = s.idx;
    const double us = uniform1(fold(mkey, 0), row, rkind);
    const double* ct = M.tab_cum_t + ((size_t)a * S + cur) * S;
    int nxt = 0;
    for (int j = 0; j < S; ++j) nxt += ct[j] < us;
    nxt = nxt < S - 1 ? nxt : S - 1;
    const double uo = uniform1(fold(mkey, 1), row, rkind);
    const double* cz = M.tab_cum_z + ((size_t)a * S + nxt) * O;
    int o = 0;
    for (int j = 0; j < O; ++j) o += cz[j] < uo;
    o = o < O - 1 ? o : O - 1;
    rew = M.tab_reward[(size_t)cur * M.action_count + a];
    const bool term = M.tab_terminal[nxt] || s.term;
    obs = term ? (u32)M.obs_arity : (u32)o;
    if (s.term) {
      rew = 0.0;
      return;
    }
    s.idx = nxt;
    s.term = term ? 1 : 0;
  }
  static __device__ __forceinline__ double heuristic(const vp_model&, const State&) { return 0.0; }
  // log Z[a, s', o] (tabular.py observation model)
  static __device__ __forceinline__ double obs_loglik(const vp_model& M, const State& s, int a, u32 obs) {
    if (obs == (u32)M.obs_arity) return s.term ? 0.0 : -INFINITY;
    if (s.term) return -INFINITY;
    return M.tab_log_z[((size_t)a * M.tab_states + s.idx) * M.tab_obs + obs];
  }
};

// ------------------------------------------------------------------ SYNTHETIC
struct __align__(16) SyntheticState {
  u64 word;
  uint32_t term;
  uint32_t pad;
};
constexpr u64 kSynAct = 0xD1B54A32D192ED03ull;
constexpr u64 kSynBranch = 0xABC98388FB8FAC03ull;
constexpr u64 kSynReward = 0x8CB92BA72F3D8DD7ull;
constexpr u64 kSynHeur = 0x9FB21C651E98DF25ull;

struct SyntheticModel {
  typedef SyntheticState State;
  static __device__ __forceinline__ void step(const vp_model& M, State& s, int a, u64 mkey, u64 row,
                                              u32& obs, double& rew, int rkind) {
    const double ut = uniform1(fold(mkey, 0), row, rkind);
    const double uo = uniform1(fold(mkey, 1), row, rkind);
    const double un = uniform1(fold(mkey, 2), row, rkind);
    const u64 w = s.word, ua = (u64)a;
    const u64 branch = (u64)(int64_t)floor(ut * (double)M.syn_branching);
    const u64 nxt = mix64(w + (ua + 1) * kSynAct + branch * kSynBranch + M.syn_salt);
    rew = unit53(mix64(w ^ (ua * kSynReward + M.syn_salt))) * 2.0 - 1.0;
    const int no = M.obs_arity;
    const int true_obs = (int)((nxt >> 17) % (u64)no);
    int noise = (int)floor(un * (double)no);
    noise = noise < no - 1 ? noise : no - 1;
    int o = uo < M.syn_obs_accuracy ? true_obs : noise;
    const bool term = s.term || (int)((nxt >> 40) % 1000ull) < M.syn_term_per_mille;
    obs = term ? (u32)no : (u32)o;
    if (s.term) {
      rew = 0.0;
      return;
    }
    s.word = nxt;
    s.term = term ? 1u : 0u;
  }
  static __device__ __forceinline__ double heuristic(const vp_model&, const State& s) {
    if (s.term) return 0.0;
    return 0.5 * unit53(mix64(s.word + kSynHeur));
  }
  // P(o) = acc [o == true] + (1 - acc) P(floor(u |O|) == o), u = k 2^-53 (oracle SyntheticModel)
  static __device__ __forceinline__ double obs_loglik(const vp_model& M, const State& s, int, u32 obs) {
    const int no = M.obs_arity;
    if (obs == (u32)no) return s.term ? 0.0 : -INFINITY;
    if (s.term) return -INFINITY;
    const int true_obs = (int)((s.word >> 17) % (u64)no);
    const double two53 = 9007199254740992.0;
    const double lo = ceil((double)obs / (double)no * two53);
    const double hi = (int)obs < no - 1 ? ceil((double)(obs + 1) / (double)no * two53) : two53;
    const double p_noise = (hi - lo) * kInv53;
    const double acc = M.syn_obs_accuracy;
    return log(acc * (double)((int)obs == true_obs) + (1.0 - acc) * p_noise);
  }
};

// ------------------------------------------------------------------ LIGHT-DARK
struct __align__(8) LightDarkState {
  double x, y;
  uint32_t term;
  uint32_t pad;
};

struct LightDarkModel {
  typedef LightDarkState State;
  static __device__ __forceinline__ int bin(const vp_model& M, double v) {
    double b = floor(v / M.ld_bin_width) + (double)(M.ld_bins / 2);
    b = b < 0.0 ? 0.0 : b;
    const double hi = (double)(M.ld_bins - 1);
    b = b > hi ? hi : b;
    return (int)b;
  }
  static __device__ __forceinline__ void step(const vp_model& M, State& s, int a, u64 mkey, u64 row,
                                              u32& obs, double& rew, int rkind) {
    // moves E, NE, N, NW, W, SW, S, SE, then DECLARE
    const int dxs[9] = {1, 1, 0, -1, -1, -1, 0, 1, 0};
    const int dys[9] = {0, 1, 1, 1, 0, -1, -1, -1, 0};
    const double nx = s.x + (double)dxs[a] * M.ld_step;
    const double ny = s.y + (double)dys[a] * M.ld_step;
    const bool declare = a == 8;
    const bool inside = s.x * s.x + s.y * s.y <= M.ld_goal_radius * M.ld_goal_radius;
    rew = declare ? (inside ? 100.0 : -100.0) : -1.0;
    const u64 nk = fold(mkey, 0);
    double z0, z1;  // rng.derive(0).normal(2): one Box-Muller pair in Philox mode
    if (rkind) {
      const double2 z = philox_normal_pair(nk, row, 1);
      z0 = z.x;
      z1 = z.y;
    } else {
      z0 = normal_j(nk, row, 1);
      z1 = normal_j(nk, row, 2);
    }
    const double sigma = M.ld_sigma0 + M.ld_sigma_slope * fabs(nx - M.ld_light_x);
    const int o = bin(M, nx + sigma * z0) * M.ld_bins + bin(M, ny + sigma * z1);
    const bool term = s.term || declare;
    obs = term ? (u32)M.obs_arity : (u32)o;
    if (s.term) {
      rew = 0.0;
      return;
    }
    s.x = nx;
    s.y = ny;
    s.term = term ? 1u : 0u;
  }
  static __device__ __forceinline__ double heuristic(const vp_model&, const State& s) {
    if (s.term) return 0.0;
    return -(fabs(s.x) + fabs(s.y));
  }
  // Bin mass of the per-axis Gaussian, border bins absorbing the tails (oracle LightDarkModel)
  static __device__ __forceinline__ double bin_mass(const vp_model& M, double center, double sigma, int b) {
    const int half = M.ld_bins / 2;
    const double den = sigma * 1.4142135623730951;
    const double chi = b == M.ld_bins - 1 ? 1.0 : 0.5 * (1.0 + erf(((b + 1 - half) * M.ld_bin_width - center) / den));
    const double clo = b == 0 ? 0.0 : 0.5 * (1.0 + erf(((b - half) * M.ld_bin_width - center) / den));
    return chi - clo;
  }
  static __device__ __forceinline__ double obs_loglik(const vp_model& M, const State& s, int, u32 obs) {
    if (obs == (u32)M.obs_arity) return s.term ? 0.0 : -INFINITY;
    if (s.term) return -INFINITY;
    const double sigma = M.ld_sigma0 + M.ld_sigma_slope * fabs(s.x - M.ld_light_x);
    return log(bin_mass(M, s.x, sigma, (int)obs / M.ld_bins) * bin_mass(M, s.y, sigma, (int)obs % M.ld_bins));
  }
};

// ------------------------------------------------------------------ NAVIGATION
// 24-byte record: occupancy bits of the unknown cells (<= 128), flat cell,
// open gate, terminal flag.
struct __align__(8) NavState {
  u64 occ0, occ1;
  int32_t pos;
  uint8_t gate, term;
  uint16_t pad;
};

struct NavigationModel {
  typedef NavState State;
  // neighbour / move order N, NE, E, SE, S, SW, W, NW; action 8 stays (navigation.py:42-47)
  static __device__ __forceinline__ int dr(int i) { return (i == 0 || i == 1 || i == 7) ? -1 : (i >= 3 && i <= 5) ? 1 : 0; }
  static __device__ __forceinline__ int dc(int i) { return (i >= 1 && i <= 3) ? 1 : (i >= 5 && i <= 7) ? -1 : 0; }

  // off-map, wall, closed gate or occupied unknown cell (navigation.py:146-162)
  static __device__ __forceinline__ bool blocked(const vp_model& M, const State& s, int r, int c) {
    if (r < 0 || r >= M.nav_h || c < 0 || c >= M.nav_w) return true;
    const int cell = r * M.nav_w + c;
    const int kind = M.nav_kind[cell];
    if (kind == 1) return true;
    if (kind == 2) return M.nav_aux[cell] != (int)s.gate;
    if (kind == 3) {
      const int u = M.nav_aux[cell];
      return ((u < 64 ? s.occ0 >> u : s.occ1 >> (u - 64)) & 1ull) != 0;
    }
    return false;
  }

  static __device__ __forceinline__ void step(const vp_model& M, State& s, int a, u64 mkey, u64 row, u32& obs,
                                              double& rew, int rkind) {
    // navigation.py:172-213
    const int r = s.pos / M.nav_w, c = s.pos % M.nav_w;
    const bool move = a != 8;
    const int k = a < 7 ? a : 7;
    const int tr = move ? r + dr(k) : r, tc = move ? c + dc(k) : c;
    const bool hit = move && blocked(M, s, tr, tc);
    const int nr = hit ? r : tr, nc = hit ? c : tc;
    const bool goal = M.nav_goal[nr * M.nav_w + nc] && move && !hit;
    const double rw = goal ? 20.0 : hit ? -1.1 : move ? -0.1 : -0.3;
    const bool term = s.term || goal;
    State nx = s;
    nx.pos = nr * M.nav_w + nc;
    // 8-bit noisy neighbour occupancy of the next cell: bit i flips when
    // rng.derive(0).uniform(8)[i] >= accuracy
    const u64 fk = fold(mkey, 0);
    u32 o = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool bit = blocked(M, nx, nr + dr(i), nc + dc(i));
      const bool flip = uniform_j(fk, row, (u64)(i + 1), rkind) >= M.nav_acc;
      o |= (u32)(bit != flip) << i;
    }
    obs = term ? (u32)M.obs_arity : o;
    if (s.term) {
      rew = 0.0;
      return;  // absorbing: the state stays
    }
    rew = rw;
    nx.term = term ? 1 : 0;
    s = nx;
  }

  static __device__ __forceinline__ double heuristic(const vp_model& M, const State& s) {
    return s.term ? 0.0 : M.nav_heur[s.pos];
  }

  // matches * log(acc) + misses * log(1 - acc) over the 8 bits (navigation.py:215-239)
  static __device__ __forceinline__ double obs_loglik(const vp_model& M, const State& s, int, u32 obs) {
    if (obs == (u32)M.obs_arity) return s.term ? 0.0 : -INFINITY;
    if (s.term) return -INFINITY;
    const int r = s.pos / M.nav_w, c = s.pos % M.nav_w;
    int hits = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) hits += blocked(M, s, r + dr(i), c + dc(i)) == (bool)((obs >> i) & 1u);
    const int miss = 8 - hits;
    return (double)hits * M.nav_log_acc + (miss > 0 ? (double)miss * M.nav_log_miss : 0.0);
  }
};

// ------------------------------------------------------------------ CROWDNAV
// 2704-byte record (crowdnav.py:33-52): robot, tracked distances at the last
// step, the emitted code, terminal flag, tracked person ids, curious bits and
// float32 person positions (x, y interleaved).  A row's record is far larger
// than a register file slice, so the planner keeps it in local memory (L1/L2)
// and the step streams over the people once.
constexpr int kCrowdPeople = 320;
constexpr int kCrowdTracked = 8;

struct __align__(8) CrowdState {
  double rx, ry;
  double prev[kCrowdTracked];
  int32_t last_code;
  uint32_t term;
  uint16_t tracked[kCrowdTracked];
  uint32_t curious[kCrowdPeople / 32];
  float px[2 * kCrowdPeople];
};

struct CrowdNavModel {
  typedef CrowdState State;
  // the planner and the SIR propagation step a row with the whole warp (people
  // split over the lanes), record in shared memory; step() below is the one-lane
  // form (vp_model_step: the environment step and the per-row parity hook)
  static constexpr bool kCoop = true;

  // j-th of the row's Box-Muller normals from precomputed row bases (rng.py:81-89)
  // (Philox mode: b1 is the normal stream's key itself, one block per normal)
  // person i's (x, y) motion normals, draws 2i+1 and 2i+2 (Philox: one Box-Muller pair)
  static __device__ __forceinline__ void normal_xy(u64 b1, u64 b2, u64 row, int i, int rk, double& zx, double& zy) {
    if (rk) {
      const double2 z = philox_normal_pair(b1, row, (u64)(i + 1));
      zx = z.x;
      zy = z.y;
    } else {
      zx = normal_at(b1, b2, row, (u64)(2 * i + 1), 0);
      zy = normal_at(b1, b2, row, (u64)(2 * i + 2), 0);
    }
  }
  static __device__ __forceinline__ double normal_at(u64 b1, u64 b2, u64 row, u64 j, int rk) {
    if (rk) return philox_normal(b1, row, j);
    const u64 h1 = mix64(b1 + j * kMixB), h2 = mix64(b2 + j * kMixB);
    const double u1 = ((double)(h1 >> 11) + 1.0) * kInv53;
    const double u2 = (double)(h2 >> 11) * kInv53;
    return sqrt(-2.0 * log(u1)) * cos(kTwoPi * u2);
  }
  static __device__ __forceinline__ double clamp(double v, double hi) { return fmin(fmax(v, 0.0), hi); }
  static __device__ __forceinline__ double dist(float x, float y, double rx, double ry) {
    const double dx = (double)x - rx, dy = (double)y - ry;
    return sqrt(dx * dx + dy * dy);
  }

  // crowdnav.py:116-174, every operation in numpy's order and precision
  // (float64 motion, float32 storage; no FMA contraction, see Makefile)
  static __device__ __forceinline__ void step(const vp_model& M, State& s, int a, u64 mkey, u64 row, u32& obs,
                                              double& rew, int rkind) {
    if (s.term) {  // absorbing: state, distances and code stay
      obs = (u32)M.obs_arity;
      rew = 0.0;
      return;
    }
    const bool yell = a == 4;  // N E S W YELL
    const double ddx = a == 1 ? 1.0 : a == 3 ? -1.0 : 0.0;
    const double ddy = a == 0 ? 1.0 : a == 2 ? -1.0 : 0.0;
    const double ry0 = s.ry + ddy;
    const bool entered = ry0 >= M.crowd_hall_d;
    const double rx = clamp(s.rx + ddx, M.crowd_hall_w), ry = clamp(ry0, M.crowd_hall_d);
    const u64 nk = fold(mkey, 0), uk = fold(mkey, 1);
    const u64 b1 = rkind ? nk : row_base(fold(nk, 101), row), b2 = rkind ? 0 : row_base(fold(nk, 211), row),
              bu = stream_base(uk, row, rkind);
    const double rad = M.crowd_collision;
    bool bumped = false;
#pragma unroll 2
    for (int i = 0; i < M.crowd_people; ++i) {
      double zx, zy;
      normal_xy(b1, b2, row, i, rkind, zx, zy);
      double x = (double)s.px[2 * i] + zx * M.crowd_noise;
      double y = (double)s.px[2 * i + 1] + zy * M.crowd_noise;
      const double dx = rx - x, dy = ry - y;
      const double d = sqrt(dx * dx + dy * dy);
      const double u = stream_uniform(bu, row, (u64)(i + 1), rkind);
      if (d < M.crowd_r_nearby && d > 1e-9 && u < M.crowd_react) {
        const bool cur = (s.curious[i >> 5] >> (i & 31)) & 1u;
        const double speed = yell ? -M.crowd_v_back : cur ? M.crowd_v_curious : -M.crowd_v_shy;
        const double dn = fmax(d, 1e-9);
        x = x + speed * (dx / dn);
        y = y + speed * (dy / dn);
      }
      const float fx = __double2float_rn(clamp(x, M.crowd_hall_w));
      const float fy = __double2float_rn(clamp(y, M.crowd_hall_d));
      s.px[2 * i] = fx;
      s.px[2 * i + 1] = fy;
      bumped |= dist(fx, fy, rx, ry) < rad;
    }
    rew = -1.0 - 25.0 * (yell ? 1.0 : 0.0) - 200.0 * (bumped ? 1.0 : 0.0) + 1000.0 * (entered ? 1.0 : 0.0);
    u32 code = 0;
    for (int k = 0; k < M.crowd_tracked; ++k) {
      const int t = s.tracked[k];
      const double td = dist(s.px[2 * t], s.px[2 * t + 1], rx, ry);
      code |= (u32)(td < s.prev[k]) << k;
      s.prev[k] = td;
    }
    s.rx = rx;
    s.ry = ry;
    s.last_code = (int32_t)code;
    s.term = entered ? 1u : 0u;
    obs = entered ? (u32)M.obs_arity : code;
  }

  // step() with the 32 lanes of a warp on ONE row whose record s is in shared
  // memory: lane j moves people j, j + 32, ...; the arithmetic of every person
  // is step()'s, so the result is bit-identical.  a, row, live are warp-uniform.
  static __device__ __forceinline__ void step_warp(const vp_model& M, State& s, int a, u64 mkey, u64 row, bool live,
                                                   u32& obs, double& rew, int rkind) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    obs = 0;
    rew = 0.0;
    if (!live) return;
    if (s.term) {
      obs = (u32)M.obs_arity;
      return;
    }
    const bool yell = a == 4;
    const double ddx = a == 1 ? 1.0 : a == 3 ? -1.0 : 0.0;
    const double ddy = a == 0 ? 1.0 : a == 2 ? -1.0 : 0.0;
    const double ry0 = s.ry + ddy;
    const bool entered = ry0 >= M.crowd_hall_d;
    const double rx = clamp(s.rx + ddx, M.crowd_hall_w), ry = clamp(ry0, M.crowd_hall_d);
    const u64 nk = fold(mkey, 0), uk = fold(mkey, 1);
    const u64 b1 = rkind ? nk : row_base(fold(nk, 101), row), b2 = rkind ? 0 : row_base(fold(nk, 211), row),
              bu = stream_base(uk, row, rkind);
    bool bumped = false;
    // squared-distance gates: sqrt is correctly rounded and monotone, so d < r can only
    // hold when s < r^2 (1 + 1e-12); outside the gate the reference's comparisons are
    // false and no sqrt is taken
    const double near2 = M.crowd_r_nearby * M.crowd_r_nearby * (1.0 + 1e-12);
    const double bump2 = M.crowd_collision * M.crowd_collision * (1.0 + 1e-12);
    for (int i = lane; i < M.crowd_people; i += 32) {
      const float2 p = reinterpret_cast<const float2*>(s.px)[i];
      double zx, zy;
      normal_xy(b1, b2, row, i, rkind, zx, zy);
      double x = (double)p.x + zx * M.crowd_noise;
      double y = (double)p.y + zy * M.crowd_noise;
      const double dx = rx - x, dy = ry - y;
      const double s2 = dx * dx + dy * dy;
      if (s2 < near2) {
        const double d = sqrt(s2);
        // the react draw only matters when both distance tests pass (pure function of row, i)
        if (d < M.crowd_r_nearby && d > 1e-9 && stream_uniform(bu, row, (u64)(i + 1), rkind) < M.crowd_react) {
          const bool cur = (s.curious[i >> 5] >> (i & 31)) & 1u;
          const double speed = yell ? -M.crowd_v_back : cur ? M.crowd_v_curious : -M.crowd_v_shy;
          const double dn = fmax(d, 1e-9);
          x = x + speed * (dx / dn);
          y = y + speed * (dy / dn);
        }
      }
      const float fx = __double2float_rn(clamp(x, M.crowd_hall_w));
      const float fy = __double2float_rn(clamp(y, M.crowd_hall_d));
      reinterpret_cast<float2*>(s.px)[i] = make_float2(fx, fy);
      const double ex = (double)fx - rx, ey = (double)fy - ry;
      const double e2 = ex * ex + ey * ey;
      bumped |= e2 < bump2 && sqrt(e2) < M.crowd_collision;
    }
    bumped = __any_sync(full, bumped);
    __syncwarp();  // every person written before the tracked ones are read
    double td = 0.0;
    bool closer = false;
    if (lane < M.crowd_tracked) {
      const int t = s.tracked[lane];
      td = dist(s.px[2 * t], s.px[2 * t + 1], rx, ry);
      closer = td < s.prev[lane];
    }
    const u32 code = __ballot_sync(full, closer);
    __syncwarp();
    if (lane < M.crowd_tracked) s.prev[lane] = td;
    if (lane == 0) {
      s.rx = rx;
      s.ry = ry;
      s.last_code = (int32_t)code;
      s.term = entered ? 1u : 0u;
    }
    __syncwarp();
    rew = -1.0 - 25.0 * (yell ? 1.0 : 0.0) - 200.0 * (bumped ? 1.0 : 0.0) + 1000.0 * (entered ? 1.0 : 0.0);
    obs = entered ? (u32)M.obs_arity : code;
  }

  // table of 1000 g^k - (1 - g^k) / (1 - g), k = max(ceil(depth - y) - 1, 0) (crowdnav.py:191-197)
  static __device__ __forceinline__ double heuristic(const vp_model& M, const State& s) {
    if (s.term) return 0.0;
    int k = (int)fmax(ceil(M.crowd_hall_d - s.ry) - 1.0, 0.0);
    k = k < M.crowd_heur_len ? k : M.crowd_heur_len - 1;
    return M.crowd_heur[k];
  }

  // deterministic observation: the code the state emitted (crowdnav.py:176-189)
  static __device__ __forceinline__ double obs_loglik(const vp_model& M, const State& s, int, u32 obs) {
    if (obs == (u32)M.obs_arity) return s.term ? 0.0 : -INFINITY;
    return (!s.term && (u32)s.last_code == obs) ? 0.0 : -INFINITY;
  }
};

}  // namespace vp

#ifdef VP_PLUGIN_SOURCE
#include "vp_plugin.cuh"  // a user ProblemModel compiled into this build (VP_MODEL_USER)
#endif
