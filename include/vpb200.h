/*
 * vpb200.h -- C ABI of the B200-native PORPP planning step.
 *
 * Drop-in boundary for the reference's planning path
 *   plan(belief, model, config, rng) -> PlanOutcome
 *   (/root/reference/pkg/src/vecpomdp/solver.py:79-113).
 * The reference is pure Python, so the "FFI a maintainer would bind" is a
 * ctypes binding of exactly these entry points; the
 * Python host package paper_2510_27191_b200 is that binding.
 *
 * Conventions
 *  - Every export returns int32 status (VP_OK = 0).  No C++ exception crosses
 *    the ABI.  Status -> Python exception mapping mirrors the reference's
 *    ValueError contract checks (core.py:73-81, tree.py:189-194,228-234,
 *    search.py:48-49,100-101, backup.py:36-37,69-70).
 *  - All array pointers are DEVICE pointers owned by the caller (PyTorch);
 *    the library never allocates in a hot call.  `stream` is a cudaStream_t.
 *  - Plain C types only; no torch types in any signature.
 */
#ifndef VPB200_H
#define VPB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPB200_ABI_VERSION 1

enum vp_status {
  VP_OK = 0,
  VP_ERR_INVALID = 1,   /* contract violation (reference raises ValueError) */
  VP_ERR_CAPACITY = 2,  /* arena / hash table too small: host grows + retries */
  VP_ERR_CUDA = 3,      /* CUDA launch / runtime error */
  VP_ERR_MODEL = 4      /* unsupported problem model kind */
};

enum vp_model_kind {
  VP_MODEL_MARS = 1,      /* envs/mars.py:44-257 (RockSample family) */
  VP_MODEL_TABULAR = 2,   /* envs/tabular.py:79-145 (Tiger et al.) */
  VP_MODEL_SYNTHETIC = 3, /* NEW: integer-hash scaling model (BASELINE config 5) */
  VP_MODEL_LIGHTDARK = 4  /* NEW: continuous-observation Light-Dark (config 4) */
};

enum vp_psi_dtype { VP_PSI_F32 = 0, VP_PSI_F64 = 1 };

/* Device descriptor of a ProblemModel (core.py:84-142).  Passed by value to
 * every kernel; constant tables live in device memory. */
typedef struct vp_model {
  int32_t kind;
  int32_t action_count;     /* |A|                                       */
  int32_t obs_arity;        /* terminal observation code = obs_arity      */
  int32_t state_bytes;      /* size of one packed device state record    */
  double discount;          /* gamma                                      */
  /* MARS */
  int32_t mars_n, mars_m, mars_ops, mars_pad;
  double mars_half_eff;
  const int8_t* mars_rock_at; /* [n*n], index x*n + y, -1 = no rock      */
  int16_t mars_rock_x[64];
  int16_t mars_rock_y[64];
  /* TABULAR */
  int32_t tab_states, tab_obs;
  const double* tab_cum_t;     /* [A*S*S] cumsum over s'                  */
  const double* tab_cum_z;     /* [A*S*O] cumsum over o                   */
  const double* tab_reward;    /* [S*A]                                   */
  const uint8_t* tab_terminal; /* [S]                                     */
  /* SYNTHETIC */
  int32_t syn_branching, syn_term_per_mille;
  double syn_obs_accuracy;
  uint64_t syn_salt;
  /* LIGHTDARK */
  double ld_step, ld_light_x, ld_goal_radius, ld_sigma0, ld_sigma_slope, ld_bin_width;
  int32_t ld_bins, ld_pad;
} vp_model;

/* Structure-of-arrays belief tree in HBM (tree.py:100-132 columns plus the
 * device-only hash indexes and backup scratch). */
typedef struct vp_tree {
  int32_t cap_beliefs, cap_actions;
  int32_t action_count;
  int32_t psi_dtype;          /* vp_psi_dtype                               */
  int32_t exact;              /* 1: numpy-order softmax/LSE (fp64 parity)   */
  int32_t psi_stride;         /* elements per PSI row (|A| padded to 16 B)  */
  uint64_t hmask_a, hmask_b;  /* hash capacity - 1 (power of two)          */
  /* belief table B + PSI */
  int32_t* b_parent_action;   /* -1 for the root                            */
  uint32_t* b_parent_obs;     /* 0xFFFFFFFF for the root                    */
  int32_t* b_depth;
  void* psi;                  /* [cap_beliefs * |A|] float or double        */
  double* b_lse;              /* cached (1/eta) log sum exp(eta PSI[b])      */
  double* b_value;            /* backup scratch V                           */
  double* b_weight;           /* backup scratch N                           */
  uint32_t* b_stamp;          /* per-(iteration, level) visit stamp         */
  uint8_t* b_flags;           /* bit 0: PSI row still equals init (lazy)    */
  /* action table A */
  int32_t* a_parent_belief;
  int32_t* a_action;
  double* a_reward;
  int32_t* a_visits;
  double* a_num;              /* backup scratch sum V*N                      */
  double* a_den;              /* backup scratch sum N                        */
  uint32_t* a_stamp;
  /* open-addressing hash indexes, 16-byte slots {u64 key; u32 id; u32 pad} */
  void* hash_a;               /* (belief << 32 | action)  -> action row     */
  void* hash_b;               /* (action row << 32 | obs) -> belief row     */
  int32_t* counters;          /* [0] n_beliefs [1] n_actions [2] overflow    */
  const double* init_prefs;   /* [|A|] initial PSI row                      */
  double* init_lse;           /* [1] LSE of the initial row (set by init)   */
  void* init_cdf;             /* [|A|] CDF of softmax(eta init) (PSI dtype) */
  double eta;
} vp_tree;

/* Per-plan row workspace (n = n_parallel rows) and per-level lists. */
typedef struct vp_work {
  int32_t n;
  int32_t max_levels;         /* capacity of the level lists (>= d_max)     */
  void* states;               /* [n * state_bytes]                          */
  int32_t* slot_a;            /* per row hash slot (bit 31: pre-existing)   */
  int32_t* slot_b;
  uint32_t* obs;
  double* reward;
  int32_t* action;
  int32_t* flist;             /* [(max_levels+1) * n] distinct beliefs/level */
  int32_t* fcount;            /* [max_levels+1]                             */
  int32_t* plist;             /* [max_levels * n] distinct action nodes/level*/
  int32_t* pcount;            /* [max_levels]                               */
  int32_t* level_base;        /* [2*(max_levels+1)] node counts per level    */
  uint64_t* scan_status;      /* [ceil(n / VP_SCAN_TILE)] look-back words   */
  uint32_t* scan_ticket;      /* [2]                                        */
  int32_t* leaf_belief;       /* [n] frontier belief per row after search   */
  double* leaf_value;         /* [n] heuristic per row after search         */
  unsigned long long* stats;  /* [8] or NULL: traffic counters summed over a plan:
                                 0 distinct beliefs/level, 1 distinct actions/level,
                                 2 PSI rows staged by the sampler, 3 sample launches,
                                 4 rows sampled, 5 new actions, 6 new beliefs */
  /* optional per-level traces (level-major, n each); NULL = off */
  int32_t* trace_action;
  uint32_t* trace_obs;
  int32_t* trace_anode;
  int32_t* trace_belief;
} vp_work;

#define VP_SCAN_TILE 128

/* One search call (search.py:86-119). */
typedef struct vp_search_args {
  uint64_t search_key;        /* it_rng.derive(1).key (solver.py:102)       */
  int32_t depth0;             /* batch.depth                                */
  int32_t d_max;
  uint32_t stamp_base;        /* unique per (plan, iteration)               */
  int32_t iteration;
  const int32_t* inject_actions; /* [d_max * n] level-major, or NULL       */
  const int32_t* start_beliefs;  /* [n] frontier at depth0, NULL = root     */
  const uint64_t* search_key_dev; /* device copy of search_key, or NULL     */
} vp_search_args;

/* A whole fixed-iteration planning step (solver.py:79-113) enqueued by one
 * call.  mode 2 (default): one persistent cooperative kernel with grid
 * barriers between phases; mode 1: one launch per phase, captured once into
 * a CUDA graph and replayed (re-captured when a pointer / size / model
 * parameter changes); mode 0: one launch per phase.  Host buffers must be
 * pinned; the caller synchronises the stream and then reads
 * out_host = {chosen action, n_beliefs, n_actions, overflow}. */
typedef struct vp_plan_args {
  int32_t iterations;          /* fixed-iteration budget (>= 1)             */
  int32_t d_max_cap;
  int32_t m;                   /* particles                                 */
  int32_t mode;                /* 0 kernels, 1 CUDA graph, 2 persistent     */
  double gamma;
  const void* particles_host;  /* [m * state_bytes] pinned, or NULL         */
  void* particles_dev;
  const double* cumw_host;     /* [m] cumsum(weights) pinned, or NULL       */
  double* cumw_dev;
  const uint64_t* keys_host;   /* [2*iterations] (draw, search) keys, pinned*/
  uint64_t* keys_dev;
  int32_t* out_host;           /* [4] pinned                                */
  int32_t* out_dev;            /* [4]                                       */
  uint64_t* timeline_dev;      /* mode 2 diagnostics: globaltimer stamp per  */
  int32_t timeline_cap;        /* phase boundary (NULL / 0 = off)           */
  int32_t pad0;
} vp_plan_args;

/* ---- library ---------------------------------------------------------- */
int32_t vp_abi_version(void);
const char* vp_status_string(int32_t status);
int32_t vp_last_cuda_error(void);
/* Layout self-description for binding checks: writes up to n int32 values
 * (sizeof vp_model/tree/work/search_args, selected offsets, slot size);
 * returns how many exist.  Host-only, no CUDA call. */
int32_t vp_abi_layout(int32_t* out, int32_t n);

/* ---- measurement -------------------------------------------------------- */
/* Kernel kinds, in order: draw, level_sample, assign_actions, accum_probe,
 * assign_beliefs, leaf, backup_leaves, backup_q, backup_v, parent_lists,
 * argmax, tree_init, rehash, plan (persistent kernel). */
#define VP_KERNEL_KINDS 14
/* on != 0: clear and start recording a CUDA-event pair around every launch. */
int32_t vp_profile_enable(int32_t on);
/* Sum recorded durations (ms) and launch counts per kind; returns #kinds. */
int32_t vp_profile_read(double* ms_by_kind, int64_t* launches_by_kind, int32_t nkinds);
/* Total kernel launches issued by this library since load. */
int64_t vp_launch_count(void);

/* ---- tree store (tree.py:100-132, 370-378) ----------------------------- */
/* Fresh tree: root row, init PSI row + LSE, empty hash indexes. */
int32_t vp_tree_init(const vp_tree* tree, void* stream);
/* Rebuild both hash indexes from the node columns (after capacity growth). */
int32_t vp_tree_rehash(const vp_tree* tree, void* stream);
/* Copy the 3 counters (n_beliefs, n_actions, overflow) to host memory. */
int32_t vp_tree_counts(const vp_tree* tree, int32_t* host_out, void* stream);

/* ---- planning step pieces ---------------------------------------------- */
/* Root-state draw (belief.py:37-44): u = uniform(draw_key, row); binary
 * search (side=right) in cum_weights[m]; gather packed particle records. */
int32_t vp_draw_root_states(const vp_model* model, const vp_work* work,
                            const void* particles, const double* cum_weights,
                            int32_t m, uint64_t draw_key, void* stream);
/* All levels of one search call (search.py:106-118) + leaf heuristic
 * accumulation (search.py:119, backup.py:44-51). */
int32_t vp_search(const vp_tree* tree, const vp_model* model, const vp_work* work,
                  const vp_search_args* args, void* stream);
/* Level-synchronous backup d = d_max..depth0+1 (backup.py:75-114). */
int32_t vp_backup(const vp_tree* tree, const vp_work* work, int32_t depth0,
                  int32_t d_max, double gamma, uint32_t stamp_base, void* stream);
int32_t vp_plan(const vp_tree* tree, const vp_model* model, const vp_work* work,
                const vp_plan_args* args, void* stream);
/* argmax of PSI[0] with lowest-id ties (solver.py:112) into out_dev[0]. */
int32_t vp_root_argmax(const vp_tree* tree, int32_t* out_dev, void* stream);

/* ---- test hooks (parity of individual kernels) ------------------------- */
int32_t vp_rng_uniform(uint64_t key, const int64_t* rows, int64_t n, int32_t k,
                       double* out, void* stream);
int32_t vp_rng_normal(uint64_t key, const int64_t* rows, int64_t n, int32_t k,
                      double* out, void* stream);
int32_t vp_model_step(const vp_model* model, void* states, const int32_t* actions,
                      uint64_t key, const int64_t* rows, int32_t n,
                      uint32_t* obs_out, double* reward_out, void* stream);
int32_t vp_model_heuristic(const vp_model* model, const void* states, int32_t n,
                           double* out, void* stream);
/* rows of PSI (f32/f64 per dtype) -> LSE per row, mode exact/fast. */
int32_t vp_lse_rows(const void* rows, int32_t dtype, int32_t exact, int32_t count,
                    int32_t width, double eta, double* out, void* stream);
/* Categorical draws from softmax(eta * rows[group[i]]) with uniforms u[i]. */
/* `lse` (fast mode): per-row LSE from vp_lse_rows, as the tree caches it. */
int32_t vp_sample_rows(const void* rows, int32_t dtype, int32_t exact, int32_t count,
                       int32_t width, double eta, const double* lse, const int32_t* group,
                       const double* u, int32_t n, int32_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VPB200_H */
