/*
 * fate.h -- C ABI of the B200-native FATE candidate scorer.
 *
 * Drop-in boundary for the reference's cost-matrix construction
 *   wfsched.planner.build_problem            (pkg/src/wfsched/planner.py:75-98)
 * and the scorer methods it calls
 *   wfsched.costs.CostModel.plan_score       (pkg/src/wfsched/costs.py:233-247)
 *   CostModel.sched_score / score_terms      (costs.py:149-231)
 *   CostModel._marginal_shard_score          (costs.py:249-279)
 *   CostModel.tail_value                     (costs.py:281-352)
 *   CostModel.realized_duration (full batch) (costs.py:383-416, consumed by
 *                                             FatePolicy._extend_work_conserving,
 *                                             policies.py:91-95)
 *
 * Plain C: pointers and sizes only, no torch types.  Every array pointer in
 * fate_bank / fate_state / fate_work / fate_windows / fate_derived / fate_out
 * is a DEVICE pointer (caller-owned, e.g. torch tensors) unless the function
 * says "host".  All launches are stream-ordered on the stream passed in
 * (cudaStream_t cast to void*; NULL = legacy default stream).
 *
 * Indexing conventions (SURVEY.md §7.1 rule 2):
 *   - stage index  = rank of the stage id in sorted(stage_ids) of its
 *                    instance, offset by fate_bank.inst_stage_off[inst]
 *                    ("global stage index");
 *   - device index = rank of the device id in sorted(device_ids);
 *   so every sorted(...) iteration of the reference is ascending-index order.
 *
 * Status codes: 0 = ok, < 0 = invalid argument (FATE_E*), > 0 = cudaError_t.
 * fate_last_error() returns a thread-local message for the last failure.
 * Arithmetic: IEEE fp64, the reference's association order, no FMA
 * contraction; results are bit-identical to CPython 3.12 running the
 * reference (whose builtin sum() is Neumaier-compensated).
 */
#ifndef FATE_H
#define FATE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FATE_ABI_VERSION 3
#define FATE_MAX_DEVICES 64
#define FATE_MAX_HORIZON 32
#define FATE_MAX_QUERIES 256
#define FATE_MAX_KAPPA 64

/* fate_weights.ablation bits (reference config.py:91-113) */
#define FATE_NO_FUTURE_PLANNING 1u
#define FATE_NO_LOCALITY 2u
#define FATE_NO_SAME_MODEL 4u
#define FATE_NO_PREFIX 8u
#define FATE_NO_SHARD 16u

/* fate_bank.flags bits */
#define FATE_BANK_UNIFORM_SPEED 1   /* every device has the same speed_factor */
#define FATE_BANK_NO_QGROUPS 2      /* no query has a prefix group (q_group all -1);
                                       lets fate_score run its lean kernel */

/* fate_bank.st_flags bits */
#define FATE_STAGE_CACHE_REUSE 1
#define FATE_STAGE_KEEP_CACHE 2

#define FATE_EINVAL (-1)
#define FATE_ETOOBIG (-2)
#define FATE_ENOTREADY (-3)

/* ScoreWeights (reference config.py:116-158) as a POD constant bank.  Host
 * memory; passed by value into the kernels' constant parameter space. */
typedef struct fate_weights {
    double lambda_q, lambda_s, lambda_tr, lambda_c, lambda_p, lambda_r;
    double gamma, kappa_prefix, locality_coeff, shard_overhead_frac, demand_coeff;
    double state_scale, locality_scale, prefix_scale, switch_x, transfer_x, prefix_x;
    /* gamma ** l for l = 0..FATE_MAX_HORIZON-1, computed on the host with
     * Python float pow (costs.py:349) */
    double gamma_pow[FATE_MAX_HORIZON];
    int32_t horizon;      /* raw weights.horizon (FatePolicy tests == 0) */
    int32_t eff_horizon;  /* weights.effective_horizon() */
    uint32_t ablation;    /* FATE_NO_* bits */
    int32_t reserved;
} fate_weights;

/* Static side: one RunConfig (devices, model catalog, role table) plus a
 * batch of workflow instances concatenated.  Device pointers. */
typedef struct fate_bank {
    int32_t n_devices;     /* D <= FATE_MAX_DEVICES */
    int32_t n_models;      /* catalog models; model ids >= n_models have no profile */
    int32_t n_roles;       /* role table rows (the neutral role included) */
    int32_t has_overrides; /* any DeviceTopology.transfer_overrides entry */
    int32_t n_instances;
    int32_t n_stages;      /* total over instances */
    int32_t n_edges;       /* total over instances */
    int32_t n_queries;     /* total over instances */
    int32_t max_queries;   /* max batch size over instances <= FATE_MAX_QUERIES */
    int32_t flags;         /* FATE_BANK_* */
    double beta_default;            /* DeviceTopology.default_transfer_coeff */
    const double* dev_speed;        /* [D] speed_factor */
    const int32_t* dev_topo_order;  /* [D] device index at topology position i */
    const double* beta;             /* [D*D] transfer_coeff(src,dst), src-major */
    const double* model_prefill;    /* [n_models] prefill_coeff */
    const double* model_decode;     /* [n_models] decode_coeff */
    const double* model_switch;     /* [n_models] switch_penalty */
    const double* role_cplx;        /* [n_roles] complexity */
    const double* role_prefill;     /* [n_roles] prefill_scale */
    const double* role_decode;      /* [n_roles] decode_scale */
    const double* role_comm;        /* [n_roles] comm_weight */
    const int32_t* inst_stage_off;  /* [I] */
    const int32_t* inst_n_stages;   /* [I] */
    const int32_t* inst_query_off;  /* [I] */
    const int32_t* inst_n_queries;  /* [I] */
    /* per stage [n_stages] */
    const int32_t* st_inst;
    const int32_t* st_model;        /* model id, -1 = None */
    const int32_t* st_role;         /* role row */
    const int32_t* st_prompt;       /* prompt_token_proxy */
    const int32_t* st_out;          /* output_token_proxy */
    const int32_t* st_group;        /* shared_prefix_group id, -1 = None */
    const int32_t* st_flags;        /* FATE_STAGE_* */
    const int32_t* st_shard;        /* shard_bound R(v) */
    const int32_t* st_level;        /* annotations.level */
    const int32_t* st_override;     /* row into override_cost, -1 = none */
    const uint64_t* st_elig;        /* eligible-device bitmask */
    /* CSR adjacency over global stage indices, rows sorted ascending */
    const int32_t* par_ptr;         /* [n_stages+1] */
    const int32_t* par_idx;         /* [n_edges] */
    const int32_t* ch_ptr;          /* [n_stages+1] */
    const int32_t* ch_idx;          /* [n_edges] */
    const double* override_cost;    /* [rows*D] base_cost_override values */
    const uint64_t* override_mask;  /* [rows] devices present in the override */
    /* queries [n_queries], instance order */
    const int32_t* q_prompt;
    const int32_t* q_group;         /* prefix group id, -1 = None */
} fate_bank;

/* Per-scenario execution-state snapshot (reference state.py:45-57 read side). */
typedef struct fate_state {
    int32_t n_scenarios;
    int32_t kappa_cap;              /* prefix entries per device <= FATE_MAX_KAPPA */
    const int32_t* scen_inst;       /* [S] instance of the scenario */
    const double* scen_clock;       /* [S] */
    const int64_t* scen_loc_off;    /* [S] offset of the instance-local loc row */
    const int32_t* scen_done_level; /* [S] max level of a stage with a located output
                                       (-1 if none): window parents above it cannot be
                                       located, so their gather is skipped */
    const int32_t* loc;             /* output_device(u) as device index, -1 = None */
    const int32_t* residency;       /* [S*D] model id, -1 = None */
    const double* dev_free;         /* [S*D] device_free */
    const int32_t* kappa_n;         /* [S*D] live prefix entries */
    const int32_t* kappa;           /* [S*D*cap*4] (group, tokens, model, 0) */
} fate_state;

/* Work list: one item = (scenario, stage) = one CTA-sized unit. */
typedef struct fate_work {
    int32_t n_items;
    int32_t reserved;
    const int32_t* scen;            /* [W] */
    const int32_t* stage;           /* [W] global stage index */
    const int64_t* psi_off;         /* [W] first psi entry of the item */
    /* optional: the work list's own ticket counter (2 x uint32, zero on
     * creation; each launch leaves it zero again).  Launches of different
     * work lists then never share a counter however many are in flight;
     * NULL = the library's rotating counters (128 direct-launch slots). */
    uint32_t* queue;
} fate_work;

/* Horizon windows: descendants of each stage bucketed by level offset
 * l = 1..levels (levels = eff_horizon-1), each bucket ascending
 * (reference costs.py:354-379). */
typedef struct fate_windows {
    int32_t levels;
    int32_t max_level_ops;          /* max over (v,l) of sum_{x in bucket}(2+|Pa(x)|) */
    const int64_t* ptr;             /* [n_stages*levels+1] */
    const int32_t* idx;             /* [ptr[end]] global stage indices */
    const int64_t* wpar_ptr;        /* [n_stages*levels+1] window parents per (v, l) */
    const int32_t* wpar_idx;        /* distinct parents != v of the bucket, ascending */
    const int32_t* wpar_minlvl;     /* [n_stages*levels] min level of those parents
                                       (INT32_MAX if none) */
} fate_windows;

/* Static per-(bank, weights) tables produced by fate_prepare. */
typedef struct fate_derived {
    double* mean_base;              /* [n_stages] CostModel._mean_base */
    double* demand;                 /* [n_stages*levels] max mean_base per bucket */
    double* split_penalty;          /* [n_stages] slot>=1 split penalty */
    double* edge_sigma;             /* [n_edges] sigma(par_idx[e] -> child) */
    double* edge_term;              /* [n_edges] tail locality term at beta_default */
    double* row_sums;               /* [n_stages*6] Neumaier sums (full batch, k=2 shard 0,
                                       shard 1) of the stateless row (stage part P) and of
                                       the full-hit row (stage part 0); valid under
                                       FATE_BANK_UNIFORM_SPEED (costs.py:257, :404-405) */
    int32_t* inst_qgroups;          /* [n_instances] 1 if any query has a prefix group */
    double* tail_sum;               /* [n_stages*(n_models+1)] full tail value per
                                       (stage, displacement class) when no level has a
                                       locality op (costs.py:281-352) */
    double* tail_static;            /* [n_stages*levels*(n_models+1)] per (stage, level,
                                       displacement class): the level's tail term
                                       gamma**l * (affinity/len(bucket) + demand_coeff *
                                       demand) with no locality op applied
                                       (costs.py:307-351); 0 for an empty bucket */
    void* stage_rec;                /* [n_stages] 112-byte stage records (static per-stage
                                       scalars of one item, csrc/fate_score_v6.cuh V6Stage) */
    int64_t* tmpl_ptr;              /* [n_stages*levels+1] op-template offsets: exclusive
                                       scan of fate_template_count's counts */
    void* tmpl;                     /* [tmpl_ptr[end]] 16-byte op-template entries: per
                                       (v, l) the reference's tail op sequence
                                       (costs.py:307-348), edge entries resolved per
                                       scenario by parent location */
    int32_t* tok_vals;              /* [n_stages*4] up to 3 partial-hit token counts t
                                       (0 < t < P(v): prompts of keep_cache stages of v's
                                       prefix group, the values state.py:236-247 seeds)
                                       and their count */
    double* tok_sums;               /* [n_stages*9] Neumaier sums (full batch, k=2 shard 0,
                                       shard 1) of the row with stage part P(v) - t, per t;
                                       valid under FATE_BANK_UNIFORM_SPEED without query
                                       prefix groups (costs.py:257, :404-405) */
} fate_derived;

/* Outputs.  psi: per item bound(v)*D entries, slot-major, NaN where the
 * device is not eligible; bound(v) = 1 if no_shard else min(R(v), |A(v)|).
 * sched/tail/completion: [W*D], NaN where not eligible; may be NULL.
 * timing: [W*D*3] (switch_s, transfer_s, compute_s) of
 * CostModel.realized_duration(stage, [(d, all queries)]) (costs.py:383-416),
 * the ShardTiming whose total_s the work-conserving fill compares
 * (policies.py:91-95); NaN where not eligible; may be NULL. */
typedef struct fate_out {
    double* psi;
    double* sched;
    double* tail;
    double* completion;
    double* timing;
} fate_out;

int fate_abi_version(void);
const char* fate_last_error(void);

/* Host: count then fill the horizon windows from HOST CSR children +
 * levels.  ptr_out has n_stages*levels+1 entries; idx_out has *n_items. */
int fate_windows_count_host(int32_t n_stages, const int32_t* ch_ptr, const int32_t* ch_idx,
                            const int32_t* level, int32_t levels, int64_t* n_items);
int fate_windows_build_host(int32_t n_stages, const int32_t* ch_ptr, const int32_t* ch_idx,
                            const int32_t* level, int32_t levels, int64_t* ptr_out,
                            int32_t* idx_out);

/* Host: distinct window parents per (v, l); call with NULL outputs to count
 * (*n_out), then with ptr_out [n_stages*levels+1] and idx_out [*n_out]. */
int fate_window_parents_host(int32_t n_stages, int32_t levels, const int64_t* win_ptr,
                             const int32_t* win_idx, const int32_t* par_ptr,
                             const int32_t* par_idx, int64_t* ptr_out, int32_t* idx_out,
                             int64_t* n_out);

/* Device: static prologue (mean_base, demand, split penalty, edge sigma and
 * locality terms).  Once per (bank, weights). */
int fate_prepare(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                 const fate_derived* out, void* stream);

/* Device: op-template length of every (stage, level) window into counts
 * [n_stages*levels] (device).  The caller scans it into fate_derived.tmpl_ptr,
 * allocates fate_derived.tmpl (16 bytes per entry) and calls fate_prepare,
 * which fills the templates and the stage records when those pointers are
 * set.  Once per (bank, weights). */
int fate_template_count(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                        const fate_derived* der, int64_t* counts, void* stream);

/* Device: score every work item.  Ψ for all slots and eligible devices, plus
 * the optional S / tail / completion matrices. */
int fate_score(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
               const fate_derived* der, const fate_state* st, const fate_work* work,
               const fate_out* out, void* stream);

/* ---- executor-side realized durations ------------------
 * CostModel.realized_duration(stage, [(device, queries)], state)
 * (costs.py:383-416) of n_tasks independent shard tasks on scenario `scen` of
 * a fate_state (e.g. the device-resident mirror of the running instance):
 * timing[3*i .. 3*i+2] = (switch_s, transfer_s, compute_s) of task i, whose
 * queries are the instance-local query indices task_queries[q0 .. q0+nq) in
 * order (compute_s is their CPython sum).  Device pointers; the caller
 * validates eligibility and disjointness (costs.py:391-401) on the host. */
typedef struct fate_task {
    int32_t stage;                  /* global stage index */
    int32_t device;
    int32_t q0;
    int32_t nq;
} fate_task;

int fate_realized(const fate_bank* bank, const fate_weights* w, const fate_state* st,
                  int32_t scen, int32_t n_tasks, const fate_task* tasks,
                  const int32_t* task_queries, double* timing, void* stream);

/* ---- host frontier solve -------------------------------
 * Native restatement of wfsched.planner.solve_frontier with its front half
 * _stage_options and the deadline fallback _greedy_fallback
 * (planner.py:101-234), same selection, objective bits, optimal flag and
 * node count.  One problem = one FrontierProblem: stages in sorted(stage_id)
 * order (only stages that have candidates), per stage its slots 0..bound-1,
 * per slot the eligible devices ascending (device index = rank in
 * sorted(device_ids)) with their Psi.  HOST memory. */
typedef struct fate_frontier {
    int32_t n_stages;
    int32_t n_devices;              /* <= FATE_MAX_DEVICES */
    const int32_t* slot_ptr;        /* [n_stages+1] into the slot rows */
    const int32_t* cand_ptr;        /* [slot_ptr[n_stages]+1] into cand_* */
    const int32_t* cand_dev;        /* device index, ascending within a slot */
    const double* cand_psi;
} fate_frontier;

typedef struct fate_selection {
    int32_t capacity;               /* entries of stage/slot/device (>= n_devices) */
    int32_t n;                      /* selected (stage, slot, device), sorted */
    int32_t* stage;
    int32_t* slot;
    int32_t* device;
    double objective;
    int32_t optimal;                /* 0: deadline hit, greedy fallback */
    int32_t reserved;
    int64_t nodes;                  /* FrontierSolution.nodes_explored */
    int64_t n_options;              /* kept options over all stages */
    double wall_s;
} fate_selection;

/* budget_s <= 0 times out at the first memo miss (the reference's zero
 * budget); max_options <= 0 means 2^26. */
int fate_solve_frontier(const fate_frontier* p, double budget_s, int64_t max_options,
                        fate_selection* out);

/* Host: budget-0 (or budgeted) solves of many independent frontiers straight
 * from a scored batch -- the per-rank "solve all instances" step of SURVEY
 * §8(e).  Problem p owns work items [item_ptr[p], item_ptr[p+1]) (one
 * (instance, scenario) frontier, items in ascending stage order), each with
 * its bound, eligibility mask and Psi row offset (fate_work.psi_off layout,
 * HOST copies).  Results: n_sel[p] selected triples at sel[(p*D + k)*3]:
 * (work item, slot, device), sorted like FrontierSolution.selected;
 * objective[p], optimal[p].  Problems are spread over n_threads host threads
 * (<= 0: all hardware threads). */
typedef struct fate_solve_batch_args {
    int32_t n_problems;
    int32_t n_devices;
    const int32_t* item_ptr;        /* [n_problems+1] */
    const int32_t* item_bound;      /* [n_items] slots per item */
    const uint64_t* item_elig;      /* [n_items] eligible-device mask */
    const int64_t* psi_off;         /* [n_items] */
    const double* psi;              /* Psi rows (fate_out.psi layout) */
    double budget_s;
    int64_t max_options;            /* <= 0: 2^26 */
    int32_t n_threads;
    int32_t reserved;
} fate_solve_batch_args;

typedef struct fate_solve_batch_out {
    int32_t* n_sel;                 /* [n_problems] */
    int32_t* sel;                   /* [n_problems*n_devices*3] */
    double* objective;              /* [n_problems] */
    int32_t* optimal;               /* [n_problems] */
    double wall_s;                  /* whole batch */
    int32_t threads;                /* threads used */
    int32_t reserved;
} fate_solve_batch_out;

int fate_solve_batch(const fate_solve_batch_args* a, fate_solve_batch_out* o);

/* ---- device-resident execution-state mirror -----------
 * One running workflow instance's scorer state kept in HBM and updated in
 * place from the executor's transitions (reference state.py:130-272), plus
 * the GPU ready set (model.py:306-319).  fate_mirror_state exposes the
 * mirror as a one-scenario fate_state that fate_score reads directly -- no
 * per-wave snapshot / pack / upload. */
#define FATE_EV_COMMIT 0    /* commit_stage(stage, slots) */
#define FATE_EV_START 1     /* on_task_start: stage, device, time = finish_time */
#define FATE_EV_COMPLETE 2  /* on_task_complete: stage, device, time = finish,
                               queries = event_queries[q0 .. q0+nq) */

typedef struct fate_event {
    int32_t kind;
    int32_t stage;                  /* global stage index */
    int32_t device;
    int32_t slots;                  /* COMMIT: total slots of the stage */
    double time;
    int32_t q0;
    int32_t nq;
} fate_event;

typedef struct fate_mirror fate_mirror;

/* bank: the device bank holding the instance; q_group_host / q_tokens_host:
 * per query of the instance its prefix group id (-1 None) and
 * group_tokens(group, prompt) (state.py:79-85), HOST; empty_model: the model
 * id the bank gives "" (entries seeded by model-less stages). */
int fate_mirror_create(const fate_bank* bank, int32_t inst, int32_t kappa_cap,
                       const int32_t* q_group_host, const int32_t* q_tokens_host,
                       int32_t empty_model, void* stream, fate_mirror** out);
int fate_mirror_destroy(fate_mirror* m);
/* Apply events (HOST arrays, in executor order) on `stream`. */
int fate_mirror_apply(fate_mirror* m, const fate_event* events, int32_t n_events,
                      const int32_t* event_queries, int32_t n_event_queries, void* stream);
/* The mirror as a one-scenario fate_state (device pointers; scenario 0). */
int fate_mirror_state(const fate_mirror* m, fate_state* out);
/* Ready stages (global indices, unordered) into out_dev (device, >= stage
 * count of the instance); *n_out (host) after a stream synchronize.  Reports
 * errors recorded by earlier applies (kappa overflow, bad event). */
int fate_mirror_ready(fate_mirror* m, int32_t* out_dev, int32_t* n_out, void* stream);

/* Device: count kernel launches issued by this library since load (for the
 * benchmark's gpu_launches evidence). */
int64_t fate_launch_count(void);

/* ---- host-buffer entry (the reference-facing call with HOST objects) ------
 * Replaces the per-wave Python loop of wfsched.planner.build_problem
 * (planner.py:75-98) for a whole batch: state and work list in HOST memory
 * (pin it for overlap), Psi / S / completion written to HOST memory.
 *
 * Host wire format: one fixed-size record per scenario (so any scenario range
 * is ONE contiguous copy), the loc rows as int8 device indices (-1 = None;
 * D <= 64 always fits: a quarter of the int32 device-side bytes over PCIe),
 * and one 16-byte record per item.
 * Scenario record, 16-byte aligned, FATE_SCEN_REC_BYTES(D, cap) bytes:
 *   [0]          double  clock               (fate_state.scen_clock)
 *   [8]          int64   loc_off             (fate_state.scen_loc_off)
 *   [16]         int32   inst                (fate_state.scen_inst)
 *   [20]         int32   done_level          (fate_state.scen_done_level)
 *   [24]         int32   reserved[2]
 *   [32]         int32   residency[D]
 *   [32+4D]      int32   kappa_n[D]
 *   [32+8D]      double  dev_free[D]
 *   [32+16D]     int32   kappa[D*cap*4]      (group, tokens, model, 0) */
#define FATE_SCEN_REC_BYTES(D, cap) (32 + 16 * (D) + 16 * (D) * (cap))

typedef struct fate_item {
    int32_t scen;
    int32_t stage;                  /* global stage index */
    int64_t psi_off;
} fate_item;

typedef struct fate_host_batch {
    int32_t n_scenarios;
    int32_t kappa_cap;
    int64_t n_loc;
    const void* scen_rec;           /* [S * FATE_SCEN_REC_BYTES(D, kappa_cap)] */
    const int8_t* loc;              /* [n_loc] output_device index, -1 = None; scenario
                                       loc_off nondecreasing */
    int32_t n_items;
    int32_t reserved;
    int64_t n_psi;                  /* entries of the Psi output */
    const fate_item* items;         /* [n_items], scenario-major, psi_off non-decreasing
                                       (equal for an item without candidates) */
} fate_host_batch;

/* Opaque per-(process, GPU) handle: its streams, events and device
 * workspaces.  Not thread-safe; one handle per caller thread. */
typedef struct fate_pipeline fate_pipeline;

int fate_pipeline_create(int device, int n_chunks, int n_streams, fate_pipeline** out);
int fate_pipeline_destroy(fate_pipeline* p);

/* Enqueue, per scenario-aligned chunk: H2D of its scenario records, loc rows
 * and items (three copies) -> unpack into the fate_state / fate_work SoA ->
 * fate_score -> D2H of Psi [, S, completion]; chunks round-robin on the
 * handle's streams so copies in both directions overlap the scoring.  Ordered
 * after the work already on `stream`; `stream` waits for all of it, so a
 * stream synchronize (or an event recorded on it) marks the host outputs
 * ready.  sched_host / completion_host may be NULL ([n_items*D] otherwise). */
int fate_pipeline_score(fate_pipeline* p, const fate_bank* bank, const fate_weights* w,
                        const fate_windows* win, const fate_derived* der,
                        const fate_host_batch* hb, double* psi_host, double* sched_host,
                        double* completion_host, void* stream);

/* The same pipeline captured once into a CUDA graph (validation, chunking and
 * workspace sizing happen here, on the host, once) and replayed per step:
 * each replay re-reads the host inputs at the captured addresses and rewrites
 * the host outputs, so callers refill the same pinned buffers between
 * replays.  Re-capture when sizes or addresses change. */
int fate_pipeline_capture(fate_pipeline* p, const fate_bank* bank, const fate_weights* w,
                          const fate_windows* win, const fate_derived* der,
                          const fate_host_batch* hb, double* psi_host, double* sched_host,
                          double* completion_host);
int fate_pipeline_replay(fate_pipeline* p, void* stream);

/* Bytes moved host->device and device->host by the last fate_pipeline_score
 * (or captured by fate_pipeline_capture: the bytes of one replay). */
int fate_pipeline_bytes(const fate_pipeline* p, int64_t* h2d, int64_t* d2h);
/* The pipeline's device Psi workspace (valid after a run; stable until a
 * larger batch regrows it): stream-ordered after the replay/score that wrote
 * it, e.g. for an NCCL all-gather of the per-rank Psi slab. */
int fate_pipeline_device_psi(const fate_pipeline* p, const double** psi_dev);

#ifdef __cplusplus
}
#endif
#endif /* FATE_H */
