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

#define VPB200_ABI_VERSION 9

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
  VP_MODEL_LIGHTDARK = 4, /* NEW: continuous-observation Light-Dark (config 4) */
  VP_MODEL_NAVIGATION = 5, /* envs/navigation.py (13x13 grid, gates, 8-bit sensor) */
  VP_MODEL_CROWDNAV = 6,   /* envs/crowdnav.py (robot through a reactive crowd) */
  VP_MODEL_USER = 7        /* a user ProblemModel compiled in as a plug-in library (core.py:84-142;
                              paper_2510_27191_b200/plugin.py, csrc/vp_plugin.cuh); only
                              plug-in builds of this library accept it */
};

enum vp_psi_dtype { VP_PSI_F32 = 0, VP_PSI_F64 = 1 };

/* Per-row random streams (vp_model.rng_kind).  SPLITMIX64 is the reference's
 * counter hash (rng.py:26-89): trees equal the reference's.  PHILOX is the fast
 * mode the north_star names: Philox4x32-10 keyed by the same derived stream
 * keys (vp_common.cuh), statistically equivalent, not the reference's trees. */
enum vp_rng_kind { VP_RNG_SPLITMIX64 = 0, VP_RNG_PHILOX = 1 };

#define VP_COUNTERS 64
#define VP_COUNTER_ACTIONS 32
#define VP_COUNTER_LIVE_B 8     /* beliefs actually created (ids below [0] may be unused) */
#define VP_COUNTER_LIVE_A 16    /* actions actually created */
#define VP_COUNTER_DONE 24      /* search blocks finished (last one advances the id extents) */
#define VP_COUNTER_DENSE 48   /* dense PSI rows handed out (fast mode), own 128-B line */
#define VP_OVERLAY_SLOTS 4    /* realised PSI cells a belief keeps inline before it gets a dense row */

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
  const double* mars_acc;     /* [(n+1)^2] check accuracy at |dx|*(n+1)+|dy|, host numpy (mars.py:136-140) */
  const double* mars_gpow;    /* [2n+2] gamma**k, host numpy (mars.py:232-240) */
  int16_t mars_rock_x[64];
  int16_t mars_rock_y[64];
  /* TABULAR */
  int32_t tab_states, tab_obs;
  const double* tab_cum_t;     /* [A*S*S] cumsum over s'                  */
  const double* tab_cum_z;     /* [A*S*O] cumsum over o                   */
  const double* tab_reward;    /* [S*A]                                   */
  const uint8_t* tab_terminal; /* [S]                                     */
  const double* tab_log_z;     /* [A*S*O] log Z (SIR likelihood)          */
  /* SYNTHETIC */
  int32_t syn_branching, syn_term_per_mille;
  double syn_obs_accuracy;
  uint64_t syn_salt;
  /* LIGHTDARK */
  double ld_step, ld_light_x, ld_goal_radius, ld_sigma0, ld_sigma_slope, ld_bin_width;
  int32_t ld_bins, ld_pad;
  /* NAVIGATION (navigation.py:62-251); tables in row-major cell order */
  int32_t nav_h, nav_w, nav_unknown, nav_pad;
  const int8_t* nav_kind;     /* [h*w] 0 free, 1 wall, 2 gate, 3 unknown    */
  const int16_t* nav_aux;     /* [h*w] gate / unknown-cell index            */
  const uint8_t* nav_goal;    /* [h*w]                                       */
  const double* nav_heur;     /* [h*w] value heuristic per cell, host numpy (navigation.py:241-251) */
  double nav_acc, nav_log_acc, nav_log_miss; /* sensor accuracy, log(acc), log(1 - acc) (host numpy) */
  /* CROWDNAV (crowdnav.py:64-241); records hold <= 320 people, <= 8 tracked */
  int32_t crowd_people, crowd_tracked;
  double crowd_hall_w, crowd_hall_d, crowd_noise, crowd_react, crowd_r_nearby;
  double crowd_v_curious, crowd_v_shy, crowd_v_back, crowd_collision;
  const double* crowd_heur;   /* [crowd_heur_len] heuristic by remaining rows k, host numpy (crowdnav.py:203-210) */
  int32_t crowd_heur_len;
  int32_t rng_kind;           /* vp_rng_kind (0: the reference's SplitMix64 streams) */
  /* USER (plug-in models): the model's parameter block, laid out as its CUDA `Params` struct */
  const void* user_params;
  int64_t user_param_bytes;
} vp_model;

/* Structure-of-arrays belief tree in HBM (tree.py:100-132 columns plus the
 * device-only hash indexes and backup scratch).
 *
 * Node ids are handed out by the device in completion order (one atomic per
 * warp), not in the reference's first-occurrence order; every node records
 * its creation key (pass << 32 | level << 24 | first row), and sorting by it
 * reproduces the reference numbering exactly (tree.py:10-12, 180-256).  The
 * host applies that permutation when it exports tables / traces, so the hot
 * path needs no ordering scan. */
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
  int32_t* b_parent_belief;   /* = a_parent_belief[b_parent_action] (backup climbs without chasing) */
  int32_t* b_parent_act;      /* = a_action[b_parent_action]                  */
  int32_t* b_depth;
  void* psi;                  /* [cap_dense * psi_stride] float or double.  Parity mode
                                 (exact): row b is belief b's row.  Fast mode: only beliefs
                                 with more than VP_OVERLAY_SLOTS action children own a dense
                                 row (b_rec.dense_row); every other belief's row is the initial
                                 row overlaid with its realised cells (tree.py:247-253,
                                 backup.py:107-108: PSI departs from init only where (b, a)
                                 was backed up) */
  double* b_lse;              /* cached (1/eta) log sum exp(eta PSI[b])      */
  double* b_value;            /* leaf heuristic sum of the current pass      */
  int32_t* b_rows;            /* rows that reached b in the current pass     */
  void* b_acc;                /* backup accumulator, 16 B {f64 sum; u32 rows done; u32 N} */
  uint32_t* b_flags;          /* parity mode: bit0 PSI row lazily == init; bit1 row not written */
  void* b_rec;                /* fast mode: [cap_beliefs] overlay record, 16-B aligned:
                                 {u32 dense_pass (0: no dense row; else the search pass that
                                 wrote it); u32 dense_row; u16 action + 1 [4] (0: empty);
                                 PSI dtype value [4]} -- 32 B (fp32) / 48 B (fp64) */
  int32_t* b_nact;            /* action children created so far: child k takes overlay slot k;
                                 child VP_OVERLAY_SLOTS makes the row dense */
  uint64_t* b_ckey;           /* creation key (canonical order)              */
  /* action table A */
  int32_t* a_parent_belief;
  int32_t* a_action;
  double* a_reward;
  int32_t* a_visits;
  int32_t* a_rows;            /* rows through the action in the current pass */
  void* a_acc;                /* backup accumulator, 16 B {f64 sum V*N; u32 rows done; u32 sum N} */
  uint64_t* a_ckey;           /* creation key (canonical order)              */
  int32_t* a_slot;            /* child index of the action within its parent (b_nact order) */
  /* open-addressing hash indexes, 16-byte slots {u64 key; u32 id; u32 pass} */
  void* hash_a;               /* (belief << 32 | action)  -> action row     */
  void* hash_b;               /* belief key (see bkey_mode) -> belief row    */
  int32_t* counters;          /* [VP_COUNTERS]: [0] belief id extent, [2] overflow, [VP_COUNTER_ACTIONS] action id
                               extent, [VP_COUNTER_LIVE_B/_A] live node counts.  A search pass numbers
                               nodes statically -- row r creating at level l takes id extent + l n + r --
                               so ids below the extents may be unused (creation key ~0) */
  const double* init_prefs;   /* [|A|] initial PSI row                      */
  double* init_lse;           /* [1] LSE of the initial row (set by init)   */
  void* init_cdf;             /* [|A|] CDF of softmax(eta init) (PSI dtype) */
  void* psi_cdf;              /* [cap_dense * psi_stride] normalised softmax CDF of each dense PSI row
                                 (fast mode), rebuilt by the backup whenever it completes the row's
                                 belief: the search reads it with one TMA copy per distinct row */
  void* dense_meta;           /* [cap_dense] {double lse, uint32 pass, pad}: a backup that changes a
                                 dense row stamps it with its pass and the row's new LSE; the CDF
                                 kernel after the backup rebuilds the stamped rows' CDFs */
  int32_t bkey_mode;          /* belief-index key: 0 = (action row << 32 | obs); 1 = (belief << 32 |
                                 action << 20 | obs), needs |A| <= 4096 and obs < 2^20 -- both
                                 claims of a level can then be issued together */
  int32_t cap_dense;          /* rows of psi                                 */
  int32_t overlay_slots;      /* VP_OVERLAY_SLOTS in fast mode, 0 in parity mode */
  int32_t init_uniform;       /* 1: every init_prefs entry is equal (the reference's uniform
                                 reference policy): overlay LSEs have a closed form */
  double eta;
} vp_tree;

/* Per-search row workspace (n = n_parallel rows, n < 2^24). */
typedef struct vp_work {
  int32_t n;
  int32_t max_levels;         /* deepest d_max this workspace serves (<= 255) */
  void* states;               /* [n * state_bytes] start states (API search) */
  int32_t* leaves;            /* [n] distinct leaf beliefs of the last search */
  int32_t* leaf_count;        /* [1]                                        */
  int32_t* leaf_belief;       /* [n] frontier belief per row after search   */
  double* leaf_value;         /* [n] heuristic per row after search         */
  unsigned long long* stats;  /* [16] or NULL: traffic counters summed over calls:
                                 0 interior beliefs backed up, 1 actions backed up,
                                 2 PSI rows staged by the sampler, 3 search launches,
                                 4 row-levels sampled, 5 new actions, 6 new beliefs,
                                 7 leaves, 8 interior beliefs whose LSE needed a full
                                 row read, 9 overlay draws (rows drawn from a belief's
                                 inline cells), 10 dense rows materialised, 11 dense rows
                                 whose CDF a backup rebuilt, 12 overlay records whose LSE
                                 needed the closed-form fallback */
  /* optional per-level traces (level-major, n each; device ids); NULL = off */
  int32_t* trace_action;
  uint32_t* trace_obs;
  int32_t* trace_anode;
  int32_t* trace_belief;
  double* trace_reward;       /* written in VP_SEARCH_TRAJECTORY mode        */
} vp_work;

/* One search call (search.py:86-119).  With `particles` set, every row first
 * draws its start state from the particle belief (belief.py:37-44, fused);
 * otherwise start states are read from work->states. */
typedef struct vp_search_args {
  uint64_t search_key;        /* it_rng.derive(1).key (solver.py:102)       */
  int32_t depth0;             /* batch.depth                                */
  int32_t d_max;
  uint32_t pass;              /* search pass number (>= 1, increasing)      */
  int32_t pad0;
  const int32_t* inject_actions; /* [d_max * n] level-major, or NULL       */
  const int32_t* start_beliefs;  /* [n] frontier at depth0, NULL = root     */
  const uint64_t* search_key_dev; /* device copy of search_key, or NULL     */
  const void* particles;      /* [m * state_bytes] or NULL                  */
  const double* cum_weights;  /* [m] cumsum of the particle weights         */
  const uint64_t* draw_key_dev; /* device copy of draw_key, or NULL         */
  uint64_t draw_key;          /* it_rng.derive(0).key (solver.py:98)        */
  int32_t m;                  /* particles                                  */
  int32_t mode;               /* vp_search_mode                             */
  int32_t row0;               /* global id of row 0 (RNG streams, creation keys); 0 unless sharded */
  int32_t pad1;
  const uint32_t* inject_obs;    /* VP_SEARCH_INSERT: [d_max * n] observations */
  const double* inject_reward;   /* VP_SEARCH_INSERT: [d_max * n] rewards      */
  const double* inject_leaf;     /* VP_SEARCH_INSERT: [n] leaf heuristic values */
} vp_search_args;

/* Search modes.  Within a pass a row's trajectory depends only on the tree as
 * it was when the pass started (PSI changes only in the backup; nodes created
 * during the pass are lazily initial), so a pass splits into a trajectory
 * phase that can be sharded over GPUs with no interaction and an insert phase
 * that replays all trajectories into each replica of the tree. */
enum vp_search_mode {
  VP_SEARCH_FUSED = 0,       /* sample, step and insert (one GPU)                       */
  VP_SEARCH_TRAJECTORY = 1,  /* sample and step rows row0..row0+n-1 against the tree
                                read-only; write trace_action/obs/reward + leaf_value */
  VP_SEARCH_INSERT = 2       /* insert the injected trajectories of all rows, no sampling */
};

/* A whole fixed-iteration planning step (solver.py:79-113) enqueued by one
 * call: per iteration one search kernel (root draw fused) and one backup
 * kernel.  mode 1 (default): captured once into a CUDA graph and replayed
 * (re-captured when a pointer / size / model parameter changes); mode 0:
 * direct launches.  Host buffers must be pinned; the caller synchronises the
 * stream and then reads out_host = {chosen action, n_beliefs, n_actions,
 * overflow}. */
typedef struct vp_plan_args {
  int32_t iterations;          /* fixed-iteration budget (>= 1)             */
  int32_t d_max_cap;
  int32_t m;                   /* particles                                 */
  int32_t mode;                /* 0 kernels, 1 CUDA graph                   */
  double gamma;                /* passes are numbered 1..iterations (fresh tree) */
  const void* particles_host;  /* [m * state_bytes] pinned, or NULL         */
  void* particles_dev;
  const double* cumw_host;     /* [m] cumsum(weights) pinned, or NULL       */
  double* cumw_dev;
  const uint64_t* keys_host;   /* [2*iterations] (draw, search) keys, pinned*/
  uint64_t* keys_dev;
  int32_t* out_host;           /* [4] pinned                                */
  int32_t* out_dev;            /* [4]                                       */
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
/* Kernel kinds, in order: draw, search, backup, tree_init, rehash, argmax, hooks, cdf_rows. */
#define VP_KERNEL_KINDS 8
/* on != 0: clear and start recording a CUDA-event pair around every launch. */
int32_t vp_profile_enable(int32_t on);
/* Sum recorded durations (ms) and launch counts per kind; returns #kinds. */
int32_t vp_profile_read(double* ms_by_kind, int64_t* launches_by_kind, int32_t nkinds);
/* Total kernel launches issued by this library since load. */
int64_t vp_launch_count(void);

/* ---- tree store (tree.py:100-132, 370-378) ----------------------------- */
/* Fresh tree: root row, init PSI row + LSE, empty hash indexes. */
int32_t vp_tree_init(const vp_tree* tree, void* stream);
/* tree->eta changed on a live tree (search.py:86 / backup.py:75 take eta per call): recompute the
 * initial row's LSE and CDF and every live row's cached LSE. */
int32_t vp_tree_set_eta(const vp_tree* tree, void* stream);
/* Rebuild the CDF row of every dense PSI row from its cached LSE (fast mode; after
 * host-level edits -- append_actions, deserialize -- that create dense rows outside a pass). */
int32_t vp_tree_build_cdfs(const vp_tree* tree, void* stream);
/* Rebuild both hash indexes from the node columns (after capacity growth). */
int32_t vp_tree_rehash(const vp_tree* tree, void* stream);
/* Copy (n_beliefs, n_actions, overflow, belief id extent, action id extent) to host
 * memory (5 x int32): live node counts and the id ranges the columns use. */
int32_t vp_tree_counts(const vp_tree* tree, int32_t* host_out, void* stream);

/* ---- planning step pieces ---------------------------------------------- */
/* Root-state draw (belief.py:37-44) into work->states: u = uniform(draw_key,
 * row); binary search (side=right) in cum_weights[m]; gather the particle. */
int32_t vp_draw_root_states(const vp_model* model, const vp_work* work,
                            const void* particles, const double* cum_weights,
                            int32_t m, uint64_t draw_key, void* stream);
/* All levels of one search call (search.py:86-119) in ONE kernel: per row and
 * level the softmax draw, G(s,a), the (b,a) and (a,o) hash claims, reward /
 * visit accumulation; then the leaf heuristic (search.py:119) and the
 * distinct-leaf list for the backup. */
int32_t vp_search(const vp_tree* tree, const vp_model* model, const vp_work* work,
                  const vp_search_args* args, void* stream);
/* Backup of the last search (backup.py:75-114) in ONE kernel: leaf means,
 * then a bottom-up completion wave -- the last child to deliver completes its
 * action (Q, PSI scatter), the last action completes its belief (LSE). */
int32_t vp_backup(const vp_tree* tree, const vp_work* work, uint32_t pass, double gamma, void* stream);
int32_t vp_plan(const vp_tree* tree, const vp_model* model, const vp_work* work,
                const vp_plan_args* args, void* stream);
/* argmax of PSI[0] with lowest-id ties (solver.py:112) into out_dev[0]. */
int32_t vp_root_argmax(const vp_tree* tree, int32_t* out_dev, void* stream);

/* ---- SIR belief update between planning steps (belief.py:47-102) ---------- */
/* Propagate the m particles through G(s, action) with the counter RNG `key`
 * (rng.derive(retry), rows 0..m-1), reweight by log P(observation | s'), and
 * normalise: cum_out = cumsum of the new weights with cum_out[m-1] = 1
 * (belief.py:50-53) -- in numpy's serial order when `exact` (bit-identical
 * resampling), else by one block-wide parallel scan.  finite_out[0] = 1 if any
 * weight is non-zero (otherwise the caller retries with the next key,
 * belief.py:86-97). */
int32_t vp_sir_weigh(const vp_model* model, const void* states, const double* weights, int32_t m, int32_t action,
                     uint32_t observation, uint64_t key, void* states_out, double* logw_scratch, double* cum_out,
                     int32_t* finite_out, int32_t exact, void* stream);
/* Systematic resampling (belief.py:47-53): out[j] = prop[first i with cum[i] > (j + u0) / m]. */
int32_t vp_sir_resample(const vp_model* model, const void* prop, const double* cum, int32_t m, double u0,
                        void* states_out, void* stream);
/* Host-level tree mutation on device ids (tree.py:180-218 append_actions: claim (belief, action),
 * reward / visit accumulation; tree.py:220-256 append_beliefs: claim (action node, observation),
 * new rows lazily == init_prefs).  `pass` (> 0, fresh per call) orders the new nodes after every
 * existing one in the canonical export; out[i] = the edge's device id (-1: capacity exceeded). */
int32_t vp_tree_append_actions(const vp_tree* tree, const int32_t* beliefs, const int32_t* actions,
                               const double* rewards, int32_t n, uint32_t pass, int32_t* out, void* stream);
int32_t vp_tree_append_beliefs(const vp_tree* tree, const int32_t* action_nodes, const uint32_t* observations,
                               int32_t n, uint32_t pass, int32_t* out, void* stream);
/* Belief reconciliation with the executed state (ProblemModel.reconcile_belief, core.py:119-136;
 * crowdnav.py:213-224): every particle record takes `source`'s bytes except [keep_lo, keep_hi)
 * (the hidden component, kept per particle).  Sizes and offsets are multiples of 8. */
int32_t vp_broadcast_record(void* records, int32_t m, int32_t record_bytes, const void* source, int32_t keep_lo,
                            int32_t keep_hi, void* stream);
/* HOST function (no CUDA): pack the reference's MarsStates (envs/mars.py:34-40: x, y (n, 2) int64,
 * rocks (n, m) bool, terminal (n,) bool; C-contiguous) into the device's 16-B MARS records
 * {x0 | y0 << 8 | x1 << 16 | y1 << 24 | terminal << 32, rock bits} at `dst` (pinned host memory
 * of an e2e planning step).  m <= 64. */
int32_t vp_pack_mars_states(const int64_t* x, const int64_t* y, const uint8_t* terminal, const uint8_t* rocks,
                            int64_t n, int32_t m, void* dst);
/* HOST function: the per-iteration keys of a fixed-iteration plan (solver.py:97-102):
 * out[2 i] = it.derive(0) (root draw), out[2 i + 1] = it.derive(1) (search), it = key.derive(i). */
int32_t vp_plan_keys(uint64_t key, int32_t iterations, uint64_t* out);

/* Latency probe: one thread follows `hops` dependent pointers next[p] (element indices) from
 * `start` with gpu-scope loads (atomic = 0: L2 round trips) or atom.add 0 (atomic = 1); out[0] =
 * ns per hop, out[1] = SM cycles per hop, out[2] = the final index. */
int32_t vp_probe_latency(const uint64_t* next, int32_t hops, int32_t atomic, uint64_t start, double* out,
                         void* stream);

/* ---- test hooks (parity of individual kernels) ------------------------- */
int32_t vp_rng_uniform(uint64_t key, const int64_t* rows, int64_t n, int32_t k,
                       double* out, void* stream);
int32_t vp_rng_normal(uint64_t key, const int64_t* rows, int64_t n, int32_t k,
                      double* out, void* stream);
/* Either stream kind (vp_rng_kind): uniforms (normal = 0) or Box-Muller
 * normals (normal = 1) of rows under `key`, k = 0 the single-draw form, else
 * k per row (rng.py:66-89 for SPLITMIX64; the Philox fast mode's streams). */
int32_t vp_rng_draws(uint64_t key, const int64_t* rows, int64_t n, int32_t k,
                     int32_t rng_kind, int32_t normal, double* out, void* stream);
/* Raw Philox4x32-10 blocks: counters [n][4], keys [n][2] -> out [n][4]
 * (known-answer / curand cross-checks of the fast mode's generator). */
int32_t vp_philox4x32_10(const uint32_t* counters, const uint32_t* keys, int64_t n,
                         uint32_t* out, void* stream);
int32_t vp_model_step(const vp_model* model, void* states, const int32_t* actions,
                      uint64_t key, const int64_t* rows, int32_t n,
                      uint32_t* obs_out, double* reward_out, void* stream);
int32_t vp_model_heuristic(const vp_model* model, const void* states, int32_t n,
                           double* out, void* stream);
/* log P(observation | next state, action) per record (ProblemModel.
 * observation_log_likelihood, core.py:96-99; the SIR reweighting term). */
int32_t vp_model_obs_loglik(const vp_model* model, const void* states, int32_t n,
                            int32_t action, uint32_t observation, double* out, void* stream);
/* 1 when this build carries a plug-in model (VP_MODEL_USER), else 0; the
 * plug-in's State record size in bytes through *state_bytes. */
int32_t vp_plugin_info(int32_t* state_bytes);
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
