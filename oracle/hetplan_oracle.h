/*
 * hetplan_oracle.h — CPU restatement of the reference planner's hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product library links or calls this;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it, and only as the checker. Each function restates the reference algorithm
 * in plain C (no reference code is copied) and cites the file:line it follows;
 * P/ = /root/reference/proj/.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference library compiled from its own sources (oracle/_ref/, see Makefile)
 * and against the committed golden vectors in tests/golden/.
 */
#ifndef HETPLAN_ORACLE_H_
#define HETPLAN_ORACLE_H_

#ifdef __cplusplus
extern "C" {
#endif

/* Grouping search statistics (the reference only exposes `visited`,
 * P/include/hetplan/grouping.hpp:64; the rest instrument the same DFS). */
typedef struct hpo_grouping_stats {
  long long visited;        /* child entries, P/src/grouping.cpp:174-178 */
  long long internal;       /* internal nodes that computed a bound (:154-160) */
  long long leaves;         /* leaves reached (:138) */
  long long feasible;       /* leaves passing (3b) and offered (:147) */
  long long bound_prunes;   /* :161-162 */
  long long deficit_prunes; /* :164-169 */
  long long improvements;   /* offers that changed best.front() */
  double model_ops;         /* fp64-op model of SURVEY.md section 8(d) */
} hpo_grouping_stats;

/* Restates solve_grouping_topk (P/src/grouping.cpp:269-335) over TP units that
 * the caller already formed (build_tp_units, :40-75). Units are given in unit
 * order; type_id/node_id are only used for the by-type / by-node seeds
 * (:206-225; first-occurrence numbering). Returns
 *   0 ok, 3 infeasible ((3b) total memory or no feasible partition), 6 invalid.
 * Outputs: out_rgs[k*n + i] for the k-th solution (k < *out_count <= top_k),
 * out_obj[k], out_z[k]; *out_optimal, stats. */
int hpo_solve_grouping(int n, const double* power, const double* memory,
                       const int* type_id, const int* node_id, int n_microbatches,
                       double min_mem, int exact_threshold, long long node_budget,
                       int top_k, int* out_count, int* out_rgs, double* out_obj,
                       double* out_z, int* out_optimal, hpo_grouping_stats* stats);

/* The four warm-start seeds and the prune floor, P/src/grouping.cpp:206-247
 * and :299-312. Returns the best seed objective (-1 if none is feasible) and
 * writes its RGS / z. */
double hpo_seed_floor(int n, const double* power, const double* memory, const int* type_id,
                      const int* node_id, int n_microbatches, double min_mem, int* out_rgs,
                      double* out_z);

/* Restates balance_workload (P/src/partition.cpp:51-110) with the profile +
 * memory model path (stage_time :33-39, memory_ok :41-47 -> estimate_memory
 * P/src/profile.cpp:226-232 with the TOTAL microbatch count).
 *   prof[s*n_bits + b] = profiled seconds for 2^b layers of stage s's type at
 *   this tp (<= 0 means the entry is missing). stage_index[s] is 1-based.
 * Returns 0 ok, 3 infeasible, 6 missing profile entry (first one in the
 * reference's evaluation order is reported in *missing_stage / *missing_layers). */
int hpo_balance_workload(int n_layers, int P, int n_bits, const double* prof,
                         const double* mem_capacity, const int* stage_index, int tp,
                         double ppb, double pab, double opt_mult, int k_total,
                         int allow_zero, int* out_layers, double* out_times,
                         double* out_bottleneck, int* missing_stage, int* missing_layers);

/* Restates estimate_stage_time (P/src/profile.cpp:180-190): ascending-bit sum. */
double hpo_stage_time(const double* prof_row, int n_bits, int layers);

/* Restates estimate_memory (P/src/profile.cpp:200-232). */
double hpo_stage_memory(int layers, int stage_index, int total_stages, int tp, double ppb,
                        double pab, double opt_mult, int k_total);

/* Restates estimate_iteration + estimate_sync (P/src/cost.cpp:29-147) for a
 * plan given as flat arrays. Groups g = 0..G-1 with stage ranges
 * [group_off[g], group_off[g+1]) into the stage arrays:
 *   stage_layers[s], stage_time[s] (compute-only, from hpo_stage_time),
 *   stage_node[s] (node of the TP unit), stage_rank0[s] (global rank of its
 *   first device), microbatches[g].
 * Outputs per group fill/steady/total/bubble and t_sync, t_star. */
void hpo_estimate_iteration(int G, const int* group_off, const int* microbatches,
                            const int* stage_layers, const double* stage_time,
                            const int* stage_node, const int* stage_rank0, int n_layers,
                            int tp, double ppb, double pab, double intra_bw,
                            double inter_bw, int sync_max, double* out_fill,
                            double* out_steady, double* out_total, double* out_bubble,
                            double* out_t_sync, double* out_t_star);

#ifdef __cplusplus
}
#endif
#endif /* HETPLAN_ORACLE_H_ */
