// vp_plugin.cuh -- a user ProblemModel as a device model (VP_MODEL_USER).
//
// The reference plans any ProblemModel subclass (core.py:84-142): step_batch,
// value_heuristic and observation_log_likelihood are Python/numpy there.  The
// device cannot call Python per row, so a user model brings those three as CUDA
// device functions; paper_2510_27191_b200/plugin.py compiles them INTO a build of
// this library (-DVP_PLUGIN_SOURCE=<file> -DVP_PLUGIN_ONLY), where the search,
// backup, SIR and plan kernels are instantiated for UserModel exactly as for the
// built-in models -- a plug-in plans at built-in speed.
//
// The user source (plugin.py: CudaModel.source) defines, inside namespace vp_user:
//   struct Params { ... };   // parameter block: the bytes of CudaModel.params
//   struct State  { ... };   // per-row record: the bytes of one CudaModel.state_dtype row
//   __device__ void step(const Params&, State& s, int a, const vp::RowDraws& rng,
//                        uint32_t& obs, double& reward);          // G(s, a), in place
//   __device__ double heuristic(const Params&, const State&);     // leaf value, 0 on terminal
//   __device__ double obs_log_likelihood(const Params&, const State& next, int a, uint32_t obs);
// A model whose record is too large for one lane (CrowdNav-sized) also defines
//   #define VP_USER_COOP 1
//   __device__ void step_warp(const Params&, State& s, int a, const RowDraws& rng, bool live,
//                             uint32_t& obs, double& reward);
// called by all 32 lanes of a warp with warp-uniform (a, rng, live) and s in shared memory;
// the lanes split the record, every lane returns the same (obs, reward), and the result must
// equal step()'s (the search and the device SIR step one row per warp with it; the
// environment step and vp_model_step use step()).
// The source is included inside namespace vp_user after the library's headers: it must
// not #include anything itself (<cstdint> types, CUDA math and the runtime are in scope).
// RowDraws is the row's BoundRng (rng.py:96-120): rng.uniform(site) is
// rng.derive(site).uniform(), rng.uniform(site, j) the j-th (1-based) of
// rng.derive(site).uniform(k), and likewise normal(); either stream kind.
#pragma once

#include "vp_common.cuh"

namespace vp {

struct RowDraws {
  u64 key, row;
  int rk;
  __device__ __forceinline__ double uniform(u64 site) const { return uniform1(fold(key, site), row, rk); }
  __device__ __forceinline__ double uniform(u64 site, u64 j) const { return uniform_j(fold(key, site), row, j, rk); }
  __device__ __forceinline__ double normal(u64 site) const { return normal_j(fold(key, site), row, 0, rk); }
  __device__ __forceinline__ double normal(u64 site, u64 j) const { return normal_j(fold(key, site), row, j, rk); }
};

}  // namespace vp

namespace vp_user {
using vp::RowDraws;
#include VP_PLUGIN_SOURCE
}  // namespace vp_user

namespace vp {

struct UserModel {
  typedef vp_user::State State;
  typedef vp_user::Params Params;
  static __device__ __forceinline__ const Params& params(const vp_model& M) {
    return *static_cast<const Params*>(M.user_params);
  }
  static __device__ __forceinline__ void step(const vp_model& M, State& s, int a, u64 mkey, u64 row, u32& obs,
                                              double& rew, int rk) {
    const RowDraws r{mkey, row, rk};
    u32 o = 0;
    double w = 0.0;
    vp_user::step(params(M), s, a, r, o, w);
    obs = o;
    rew = w;
  }
#ifdef VP_USER_COOP
  static constexpr bool kCoop = true;
  static __device__ __forceinline__ void step_warp(const vp_model& M, State& s, int a, u64 mkey, u64 row, bool live,
                                                   u32& obs, double& rew, int rk) {
    obs = 0;
    rew = 0.0;
    if (!live) return;
    const RowDraws r{mkey, row, rk};
    u32 o = 0;
    double w = 0.0;
    vp_user::step_warp(params(M), s, a, r, live, o, w);
    obs = o;
    rew = w;
  }
#endif
  static __device__ __forceinline__ double heuristic(const vp_model& M, const State& s) {
    return vp_user::heuristic(params(M), s);
  }
  static __device__ __forceinline__ double obs_loglik(const vp_model& M, const State& s, int a, u32 obs) {
    return vp_user::obs_log_likelihood(params(M), s, a, obs);
  }
};

}  // namespace vp
