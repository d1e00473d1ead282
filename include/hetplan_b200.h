/*
 * hetplan_b200.h — drop-in boundary of the B200-native plan search.
 *
 * 1. The library (paper_2512_20953_b200/libhetplan_b200.so) exports the
 *    reference C ABI of P/include/hetplan/c_api.h UNCHANGED (P = the
 *    reference project, /root/reference/proj). The entry point whose
 *    implementation is replaced is
 *
 *      hp_status hp_plan_compute(const hp_cluster*, const hp_model*,
 *                                const hp_profile*, const hp_plan_options*,
 *                                hp_plan** out);            (c_api.h:91-93)
 *
 *    which calls hetplan::plan_cluster (P/src/c_api.cpp:205-206); that one
 *    translation unit (P/src/planner.cpp) is replaced by
 *    paper_2512_20953_b200/csrc/planner_b200.cpp, which drives the sm_100a
 *    kernels below. Every other hp_* symbol keeps the reference's behaviour
 *    (CLI/IO, simulator, checkpoint, recovery are the reference's own code).
 *    The hp_* prototypes are repeated here, each citing the reference
 *    declaration it is bound to, so that the boundary is self-describing.
 *
 * 2. The thin kernel C-ABI (hpk_*) that planner_b200.cpp calls: plain
 *    pointers and sizes, no C++ or torch types, no exceptions across it.
 *    Return value 0 = success; otherwise an hp_status-compatible code and
 *    hpk_last_error() (thread-local) describes it.
 */
#ifndef HETPLAN_B200_H_
#define HETPLAN_B200_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ *
 * Reference C ABI, exported unchanged (P/include/hetplan/c_api.h)     *
 * ------------------------------------------------------------------ */
typedef struct hp_cluster hp_cluster;       /* c_api.h:33 */
typedef struct hp_model hp_model;           /* c_api.h:34 */
typedef struct hp_profile hp_profile;       /* c_api.h:35 */
typedef struct hp_plan hp_plan;             /* c_api.h:36 */
typedef struct hp_sim_result hp_sim_result; /* c_api.h:37 */
typedef struct hp_recovery hp_recovery;     /* c_api.h:38 */

typedef enum hp_status { /* c_api.h:41-48: values double as CLI exit codes */
  HP_OK = 0,
  HP_PARSE_ERROR = 2,
  HP_INFEASIBLE = 3,
  HP_UNRECOVERABLE = 4,
  HP_INTERNAL_ERROR = 5,
  HP_INVALID_ARGUMENT = 6
} hp_status;

typedef struct hp_plan_options { /* c_api.h:76-87, field for field */
  const int* tp_dims;
  int n_tp_dims;
  double min_mem_override;
  int exact_threshold;
  long long node_budget;
  int top_k;
  int sync_overlap_max;
  int validate_with_sim;
  int derive_power;
  const char* power_reference;
} hp_plan_options;

typedef struct hp_sim_options { /* c_api.h:105-109 */
  int combined_time;
  double fb_ratio;
  int zero_comm;
} hp_sim_options;

const char* hp_version(void);                                         /* c_api.h:50 */
const char* hp_last_error(void);                                      /* c_api.h:51 */
void hp_string_free(char* s);                                         /* c_api.h:52 */
hp_status hp_cluster_load_file(const char* path, hp_cluster** out);   /* c_api.h:55 */
hp_status hp_cluster_parse(const char* text, hp_cluster** out);       /* c_api.h:56 */
int hp_cluster_device_count(const hp_cluster* cluster);               /* c_api.h:57 */
hp_status hp_cluster_warnings(const hp_cluster* cluster, char** out); /* c_api.h:59 */
void hp_cluster_free(hp_cluster* cluster);                            /* c_api.h:60 */
hp_status hp_model_load_file(const char* path, hp_model** out);       /* c_api.h:63 */
hp_status hp_model_parse(const char* text, hp_model** out);           /* c_api.h:64 */
void hp_model_free(hp_model* model);                                  /* c_api.h:65 */
hp_status hp_profile_load_file(const char* path, hp_profile** out);   /* c_api.h:68 */
hp_status hp_profile_parse(const char* text, hp_profile** out);       /* c_api.h:69 */
hp_status hp_profile_synth(const hp_cluster* cluster, double base_seconds_per_layer,
                           int max_layers, hp_profile** out);         /* c_api.h:70-71 */
hp_status hp_profile_write_file(const hp_profile* profile, const char* path); /* c_api.h:72 */
void hp_profile_free(hp_profile* profile);                            /* c_api.h:73 */
void hp_plan_options_init(hp_plan_options* options);                  /* c_api.h:89 */
/* THE replaced entry point: plan search on the B200 (c_api.h:91-93). */
hp_status hp_plan_compute(const hp_cluster* cluster, const hp_model* model,
                          const hp_profile* profile, const hp_plan_options* options,
                          hp_plan** out);
/* Extension (not in the reference ABI): hp_plan_compute over n clusters that
 * share a model — e.g. the snapshots of a spot-preemption replanning sweep
 * (SURVEY.md 8(d) cfg5). Every cluster's TP-dimension searches go into ONE
 * grouping-search launch and every candidate into ONE partition/cost launch;
 * the host phases (unit formation, stage mapping, selection) run on
 * host_threads threads (<= 0: all cores). out_plans[i] / out_status[i] are
 * what hp_plan_compute returns for cluster i; out_errors[i] (optional) is its
 * error message or NULL (free with hp_string_free). Returns HP_OK unless an
 * argument is invalid. Results equal n hp_plan_compute calls byte for byte. */
hp_status hp_plan_compute_batch(int n, const hp_cluster* const* clusters, const hp_model* model,
                                const hp_profile* const* profiles,
                                const hp_plan_options* options, int host_threads,
                                hp_plan** out_plans, hp_status* out_status, char** out_errors);
hp_status hp_plan_load_file(const char* path, hp_plan** out);         /* c_api.h:94 */
hp_status hp_plan_write_file(const hp_plan* plan, const char* path);  /* c_api.h:95 */
hp_status hp_plan_to_json(const hp_plan* plan, char** out);           /* c_api.h:96 */
hp_status hp_plan_explain(const hp_plan* plan, char** out);           /* c_api.h:97 */
void hp_plan_free(hp_plan* plan);                                     /* c_api.h:98 */
hp_status hp_estimate_to_json(const hp_plan* plan, const hp_cluster* cluster,
                              const hp_model* model, const hp_profile* profile,
                              char** out);                            /* c_api.h:101-103 */
void hp_sim_options_init(hp_sim_options* options);                    /* c_api.h:111 */
hp_status hp_simulate(const hp_plan* plan, const hp_cluster* cluster, const hp_model* model,
                      const hp_profile* profile, const hp_sim_options* options,
                      hp_sim_result** out);                           /* c_api.h:113-115 */
double hp_sim_makespan(const hp_sim_result* result);                  /* c_api.h:116 */
hp_status hp_sim_result_to_json(const hp_sim_result* result, char** out); /* c_api.h:117 */
hp_status hp_sim_timeline_csv(const hp_sim_result* result, char** out);   /* c_api.h:119 */
void hp_sim_result_free(hp_sim_result* result);                       /* c_api.h:120 */
hp_status hp_checkpoint_save(const hp_plan* plan, const char* root, unsigned long long step,
                             int hidden_dim, unsigned long long seed,
                             int zero_optimizer);                     /* c_api.h:123-125 */
hp_status hp_recovery_compute(const hp_plan* old_plan, const hp_plan* new_plan,
                              const char* bitmap_path, const hp_cluster* cluster,
                              hp_recovery** out);                     /* c_api.h:127-129 */
hp_status hp_recovery_load_file(const char* path, hp_recovery** out); /* c_api.h:130 */
hp_status hp_recovery_write_file(const hp_recovery* recovery, const char* path); /* c_api.h:131 */
hp_status hp_recovery_to_json(const hp_recovery* recovery, char** out);          /* c_api.h:132 */
hp_status hp_recovery_execute(const hp_recovery* recovery, const char* root,
                              const char* out_dir);                   /* c_api.h:134-135 */
void hp_recovery_free(hp_recovery* recovery);                         /* c_api.h:136 */

/* ------------------------------------------------------------------ *
 * B200 kernel C-ABI (new)                                              *
 * ------------------------------------------------------------------ */
#define HPK_MAX_UNITS 128 /* wave engine (<= 64 groups per node); larger: serial replica */
#define HPK_MAX_TOPK 16 /* wave engine (larger top_k: serial replica) */
#ifndef HPK_HOST_TRACE
#define HPK_HOST_TRACE 0 /* build with -DHPK_HOST_TRACE=1 for per-phase host timings */
#endif

const char* hpk_version(void);
const char* hpk_last_error(void); /* thread-local, valid until the next hpk_* call */
int hpk_device_count(void);       /* CUDA devices visible (0: the planner fails loudly) */

/* One DP-grouping problem: solve_grouping_topk over already-formed TP units
 * (P/src/grouping.cpp:269-335; units from build_tp_units :40-75). */
typedef struct hpk_grouping_problem {
  int n;                 /* TP units */
  int n_microbatches;    /* total K (planner.cpp:150) */
  double min_mem;        /* MIN_mem (planner.cpp:151-152) */
  int exact_threshold;   /* exhaustive iff n <= exact_threshold (grouping.cpp:296) */
  long long node_budget; /* visits beyond the threshold (grouping.cpp:174-177) */
  int top_k;             /* >= 1 */
  const double* power;   /* [n] unit powers, unit order */
  const double* memory;  /* [n] unit memories */
  const int* type_key;   /* [n] equal keys <=> same GPU type (seed by_type, :213-222) */
  const int* node_key;   /* [n] node ids (seed by_node) */
} hpk_grouping_problem;

typedef struct hpk_grouping_result {
  int status;                        /* 0 ok, 3 infeasible ((3b): no feasible partition) */
  int count;                         /* solutions (<= top_k), best first */
  int optimal;                       /* 0 if the node budget ran out (grouping.cpp:317) */
  int engine;                        /* 0 wave engine, 1 serial replica, 2 enumeration */
  long long visited;                 /* GroupingSolution::nodes_visited */
  double* objective;                 /* caller-owned [top_k] */
  double* z;                         /* caller-owned [top_k] */
  int* rgs;                          /* caller-owned [top_k * n]: group of unit i */
  /* engine statistics */
  int waves;
  long long segment_runs;
  long long segment_visits;          /* visits executed incl. speculation */
  int max_list;
  long long exact_checks;            /* child checks inside the filter margin (exact path) */
} hpk_grouping_result;

#define HPK_ALL_DEVICES (-2) /* batches worth < ~100 K budgeted visits stay on device 0 */
typedef struct hpk_search_config {
  int device;            /* CUDA ordinal (-1: current; HPK_ALL_DEVICES: every visible
                            device, problems longest-first to the least-loaded one) */
  long long segment_cap; /* visits per segment run per wave (0: default) */
  int max_list;          /* segment list capacity per problem (0: default) */
  int force_serial;      /* 1: use the serial replica kernel for every problem */
  int enumerate;         /* 1: exhaustive top_k = 1 problems with n <= 12 take the
                            enumeration engine (engine 2: winner only, visited = -1) */
  int max_waves;         /* watchdog on the wave loop (0: default 1000000) */
  double max_seconds;    /* device wall-clock watchdog (0: derived from the budgets) */
  int max_ctas;          /* wave-engine grid cap (0: every SM, 2 CTAs each) */
  int cut_intervals;     /* runs are accepted for any exact entering cutoff in their
                            recorded interval: -1 auto (launches of at
                            most 16 searches), 0 off (exact-cutoff rule), 1 on */
} hpk_search_config;

void hpk_search_config_init(hpk_search_config* cfg);

/* The device assignment HPK_ALL_DEVICES uses (host only, no CUDA call):
 * problems in decreasing estimated cost (budgeted: node_budget visits,
 * exhaustive: Bell(n), weighted by n + 8; ties in caller order) each to the
 * device with the least assigned cost (ties: lowest ordinal). */
int hpk_assign_devices(const hpk_grouping_problem* problems, int n_problems, int n_devices,
                       int* out_device);

/* Batched grouping search: every problem is searched concurrently on the GPU
 * (one persistent cooperative kernel for the wave engine). */
int hpk_grouping_search(const hpk_grouping_problem* problems, int n_problems,
                        hpk_grouping_result* results, const hpk_search_config* cfg);

/* One assembled candidate plan: layer partition (P/src/partition.cpp:51-110)
 * per DP group, then the Eq. (1) cost (P/src/cost.cpp:29-147). */
typedef struct hpk_plan_candidate {
  int n_layers, tp, k_total, n_groups;
  double ppb, pab, opt_mult; /* MemoryModel coefficients (memory check, profile.cpp:200-215) */
  double cost_ppb, cost_pab; /* ModelConfig bytes (ring volume cost.cpp:79, boundary :38) */
  double intra_bw, inter_bw; /* ClusterSpec link classes (cluster.cpp:187-192) */
  int sync_max;              /* SyncOverlap::max */
  int allow_zero;            /* PlannerOptions::allow_zero_layer_stages */
  const int* group_stage_off;        /* [n_groups+1] */
  const int* microbatches;           /* [n_groups] split_microbatches (plan.cpp:53-62) */
  const int* stage_type;             /* [n_stages] row into prof */
  const int* stage_index;            /* [n_stages] 1-based */
  const double* stage_mem_capacity;  /* [n_stages] GpuType memory */
  const int* stage_node;             /* [n_stages] node of the TP unit */
  const int* stage_rank0;            /* [n_stages] global rank of devices.front() */
  int n_types, n_bits;
  const double* prof;                /* [n_types*n_bits] seconds for 2^b layers (<=0 missing) */
} hpk_plan_candidate;

typedef struct hpk_plan_result {
  int status;          /* 0 ok, 3 infeasible, 6 missing profile entry */
  int fail_group;      /* first group that failed */
  int fail_kind;       /* 1: n_layers < stages, 2: no split fits memory */
  int missing_stage;   /* status 6: stage (global index) and layer count */
  int missing_layers;
  int* stage_layers;   /* caller-owned [n_stages] */
  double* stage_time;  /* [n_stages] compute-only stage time (StagePlan::est_time_s) */
  double* stage_mem;   /* [n_stages] estimate_memory with total K */
  double* group_fill;  /* [n_groups] GroupCost fields */
  double* group_steady;
  double* group_total;
  double* group_bubble;
  double t_sync, t_star;
} hpk_plan_result;

int hpk_partition_cost(const hpk_plan_candidate* cands, int n_cands, hpk_plan_result* results,
                       int device);

/* Same, with test hooks that force the kernel's slow branches on any input:
 * the DP's best tables in global memory instead of shared memory, and the
 * per-layer-count memory check instead of the feasible-prefix fast path. */
#define HPK_PART_GMEM_TABLES 1
#define HPK_PART_PER_L_MEMORY 2
int hpk_partition_cost_ex(const hpk_plan_candidate* cands, int n_cands,
                          hpk_plan_result* results, int device, int flags);

/* The DP-affinity pass of the stage mapper (map_nodes_and_stages,
 * P/src/stage_map.cpp:188-214) for one candidate plan: slots in stage order
 * per group after the joint / fallback placement (:94-186), each holding the
 * unit of type slot_type[s] on node slot_node[s]. The first strictly
 * improving same-type swap in (group, slot, group, slot) scan order is applied
 * until none is left (count_intra_node_dp_pairs, :39-58). On return
 * slot_perm[s] is the index of the original slot whose unit now sits in s. */
typedef struct hpk_affinity_problem {
  int n_groups, n_slots;
  const int* group_off;  /* [n_groups+1] slot offsets */
  const int* slot_type;  /* [n_slots] dense type ids */
  const int* slot_node;  /* [n_slots] node id of the slot's unit */
  int* slot_perm;        /* [n_slots] out (caller-owned) */
  int swaps;             /* out: swaps applied */
} hpk_affinity_problem;

/* All problems in one launch (one CTA each). */
int hpk_stage_affinity(hpk_affinity_problem* problems, int n_problems, int device);

/* The planner's fused launch: candidate k's affinity pass (affinity[k]), then
 * its partition + cost (cands[k]) in the same CTA, with stage_node /
 * stage_rank0 given in the PRE-affinity slot order — the kernel permutes them
 * (swaps exchange same-type units, so types, indices and capacities do not
 * change). affinity[k].n_slots must equal cands[k]'s stage count. One H2D copy,
 * one launch, one D2H copy for the whole batch. */
int hpk_affinity_partition_cost(hpk_affinity_problem* affinity, const hpk_plan_candidate* cands,
                                int n_cands, hpk_plan_result* results, int device);

/* The planner's whole stage mapping (map_nodes_and_stages,
 * P/src/stage_map.cpp:63-216) for n_groupings groupings of one cluster's TP
 * units at tp, exactly as hp_plan_compute runs it: the joint / fallback
 * placement on the host, then ONE hpk_stage_affinity launch for all of them.
 * Units are the planner's own (R2) at the GPU types' powers; grouping g puts
 * unit u in group rgs[g*U + u]. Writes the unit index of every stage slot
 * (groups in order, stages in order) to out_unit[g*U + s]. Returns U (> 0), or
 * -(hp_status) on an error (text in hpk_last_error()). Used by the parity tests
 * against the reference mapper. */
int hpk_map_stages(const hp_cluster* cluster, int tp, int n_groupings, const int* rgs,
                   int* out_unit);

/* The 1F1B schedule recurrence of simulate_pipeline (P/src/pipeline_sim.cpp:46-149)
 * for many pipelines in one launch (one CTA per pipeline, one thread per
 * stage). Inputs are the StageTiming fields per stage; outputs are the
 * reference's PipelineSimResult values: makespan, busy and peak_in_flight per
 * stage, and each stage's tasks' start / end times in the stage's static order
 * (warmup forwards, F/B pairs, backward drain; :53-66). */
typedef struct hpk_pipeline {
  int n_stages, n_microbatches;
  const double* forward;        /* [n_stages] */
  const double* backward;
  const double* send_forward;
  const double* send_backward;
  double makespan;              /* out */
  double* busy;                 /* out [n_stages] */
  int* peak_in_flight;          /* out [n_stages] */
  double* task_start;           /* out [n_stages * 2 * n_microbatches] or NULL */
  double* task_end;
} hpk_pipeline;
int hpk_pipeline_sim(hpk_pipeline* pipes, int n_pipes, int device);

/* Extension of the drop-in ABI: hp_simulate (c_api.h:113-115) for n plans of
 * one model in ONE simulator launch (every DP group of every plan). Results are
 * the reference's hp_sim_result handles (hp_sim_result_to_json /
 * hp_sim_timeline_csv / hp_sim_result_free apply). Returns the first error
 * (text in hpk_last_error()); out[i] is NULL then. */
hp_status hp_simulate_batch(int n, const hp_plan* const* plans, const hp_cluster* const* clusters,
                            const hp_model* model, const hp_profile* const* profiles,
                            const hp_sim_options* options, hp_sim_result** out);

/* Device-side timing of this thread's last hpk_grouping_search /
 * hpk_partition_cost calls (CUDA events on the launching stream). */
typedef struct hpk_timing {
  double search_ms;     /* wave-engine kernel(s) */
  double serial_ms;     /* serial replica kernel */
  double partition_ms;  /* partition + cost kernel */
  double h2d_ms, d2h_ms;
  long long h2d_bytes, d2h_bytes;
  int kernel_launches;
  int devices_used;     /* GPUs the grouping search ran on */
  double affinity_ms;   /* stage-mapper affinity kernel */
  double pipeline_ms;   /* 1F1B pipeline simulator kernel */
} hpk_timing;
void hpk_last_timing(hpk_timing* out);
void hpk_reset_timing(void);

/* Device self-test of the grouping filter decision (regression pin for an
 * nvcc 12.9 sm_100a miscompile): cases = n (A, D, cut) triplets,
 * rem = rm4[2]; writes 0 pass / 1 prune / 2 exact per case. */
int hpk_selftest_decide(const double* cases, int n, const double* rm4, double mb_abs,
                        double md_abs, int* out_codes);

/* Issue-rate microbenchmarks (roofline denominators for this FP64/INT32-issue
 * bound path): fp64 DMUL+DADD ops/s and int32 IADD+LOP ops/s on `device`. */
int hpk_measure_issue_peaks(int device, double* fp64_ops_per_s, double* int_ops_per_s);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* HETPLAN_B200_H_ */
