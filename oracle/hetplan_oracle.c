/*
 * hetplan_oracle.c — CPU restatement of the reference planner's hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see hetplan_oracle.h). Built into
 * oracle/_ref/libhpo.so by oracle/Makefile with -ffp-contract=off so every
 * fp64 operation rounds exactly where the reference's does (the reference is
 * built without -march, i.e. without FMA).
 */
#include "hetplan_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define HPO_MAX_UNITS 256

/* ---------------------------------------------------------------- grouping */

typedef struct cand {
  double objective;
  int n_groups;
  double z;
  int rgs[HPO_MAX_UNITS];
} cand;

typedef struct search {
  int n;
  const double* power;
  const double* memory;
  int k_total;
  double min_mem;
  int top_k;
  long long budget; /* < 0: unlimited */
  int aborted;
  /* per active group, P/src/grouping.cpp:88-92 */
  int G;
  double gpow[HPO_MAX_UNITS];
  double gmem[HPO_MAX_UNITS];
  int gcnt[HPO_MAX_UNITS];
  int rgs[HPO_MAX_UNITS];
  cand* best; /* best-first, at most top_k (:100) */
  int n_best;
  double prune_floor; /* :101 */
  hpo_grouping_stats st;
} search;

/* Eq. (2) group factor: P/src/grouping.cpp:103-108 (and :35-37). */
static double group_effective(const search* s, int gi) {
  const int depth = s->gcnt[gi];
  const double rho = (double)(depth - 1) / (double)(s->k_total + depth - 1);
  return s->gpow[gi] * (1.0 - rho);
}

/* Ranking, P/src/grouping.cpp:112-115: higher objective, then fewer groups. */
static int better(double ao, int ag, double bo, int bg) {
  if (ao != bo) return ao > bo;
  return ag < bg;
}

/* P/src/grouping.cpp:117-127: upper_bound insert (after equals), RGS dedup,
 * truncate to top_k. */
static void offer(search* s, double objective, double z) {
  int pos = s->n_best;
  for (int i = 0; i < s->n_best; ++i) {
    if (better(objective, s->G, s->best[i].objective, s->best[i].n_groups)) {
      pos = i;
      break;
    }
  }
  for (int i = 0; i < s->n_best; ++i) {
    if (memcmp(s->best[i].rgs, s->rgs, sizeof(int) * (size_t)s->n) == 0) return;
  }
  int cap = s->n_best + 1;
  for (int i = cap - 1; i > pos; --i) s->best[i] = s->best[i - 1];
  s->best[pos].objective = objective;
  s->best[pos].n_groups = s->G;
  s->best[pos].z = z;
  memcpy(s->best[pos].rgs, s->rgs, sizeof(int) * (size_t)s->n);
  s->n_best = cap > s->top_k ? s->top_k : cap;
  if (pos == 0) s->st.improvements++;
}

/* P/src/grouping.cpp:129-132. */
static double kth_objective(const search* s) {
  if (s->n_best < s->top_k) return s->prune_floor;
  const double b = s->best[s->n_best - 1].objective;
  return s->prune_floor > b ? s->prune_floor : b;
}

/* The DFS of P/src/grouping.cpp:135-202, statement by statement. */
static void dfs(search* s, int next) {
  if (s->aborted) return;
  const int n = s->n;
  if (next == n) { /* leaf, :138-149 */
    s->st.leaves++;
    s->st.model_ops += 3.0 * s->G + 1.0;
    double z = 0;
    int first = 1;
    for (int gi = 0; gi < s->G; ++gi) {
      if (s->gmem[gi] < s->min_mem) return; /* (3b) */
      const double g = group_effective(s, gi);
      z = first ? g : (g < z ? g : z); /* std::min(z, g) */
      first = 0;
    }
    s->st.feasible++;
    offer(s, (double)s->G * z, z);
    return;
  }
  s->st.internal++;
  const int r = n - next;
  s->st.model_ops += 2.0 * s->G + 2.0 * r + 1.0;
  /* bound, :154-160: group terms first, then remaining raw powers, serially */
  double bound = 0;
  for (int gi = 0; gi < s->G; ++gi) bound += group_effective(s, gi);
  double remaining_mem = 0;
  for (int i = next; i < n; ++i) {
    bound += s->power[i];
    remaining_mem += s->memory[i];
  }
  const double cutoff = kth_objective(s);
  if (cutoff >= 0 && bound < cutoff) {
    s->st.bound_prunes++;
    return;
  }
  s->st.model_ops += 3.0 * s->G + 1.0;
  /* memory deficit, :164-169 */
  double deficit = 0;
  for (int gi = 0; gi < s->G; ++gi) {
    const double d = s->min_mem - s->gmem[gi];
    deficit += d > 0.0 ? d : 0.0; /* std::max(0.0, d) */
  }
  if (deficit > remaining_mem) {
    s->st.deficit_prunes++;
    return;
  }
  const double up = s->power[next];
  const double um = s->memory[next];
  const int n_groups = s->G;
  for (int gi = 0; gi <= n_groups; ++gi) { /* :173-201 */
    if (s->budget >= 0 && s->st.visited >= s->budget) {
      s->aborted = 1;
      return;
    }
    ++s->st.visited;
    s->st.model_ops += 4.0;
    if (gi == n_groups) {
      s->gpow[s->G] = up;
      s->gmem[s->G] = um;
      s->gcnt[s->G] = 1;
      s->G++;
    } else {
      s->gpow[gi] += up;
      s->gmem[gi] += um;
      s->gcnt[gi] += 1;
    }
    s->rgs[next] = gi;
    dfs(s, next + 1);
    if (gi == n_groups) {
      s->G--;
    } else {
      s->gpow[gi] -= up;
      s->gmem[gi] -= um;
      s->gcnt[gi] -= 1;
    }
    if (s->aborted) return;
  }
}

/* evaluate_partition, P/src/grouping.cpp:227-247 (fresh sums, unit order). */
static double evaluate_partition(int n, const double* power, const double* memory,
                                 const int* rgs, int k_total, double min_mem, double* z_out) {
  int m = 0;
  for (int i = 0; i < n; ++i) m = rgs[i] + 1 > m ? rgs[i] + 1 : m;
  double pw[HPO_MAX_UNITS], me[HPO_MAX_UNITS];
  int cnt[HPO_MAX_UNITS];
  for (int g = 0; g < m; ++g) {
    pw[g] = 0;
    me[g] = 0;
    cnt[g] = 0;
  }
  for (int i = 0; i < n; ++i) {
    pw[rgs[i]] += power[i];
    me[rgs[i]] += memory[i];
    cnt[rgs[i]] += 1;
  }
  double z = 0;
  for (int gi = 0; gi < m; ++gi) {
    if (cnt[gi] == 0 || me[gi] < min_mem) return -1;
    const double rho = (double)(cnt[gi] - 1) / (double)(k_total + cnt[gi] - 1);
    const double g = pw[gi] * (1.0 - rho);
    z = gi == 0 ? g : (g < z ? g : z);
  }
  if (z_out) *z_out = z;
  return m * z;
}

/* First-occurrence numbering used by seed_partitions (std::map::emplace with
 * index = current size), P/src/grouping.cpp:213-221. */
static void first_occurrence(int n, const int* key, int* out) {
  int seen_key[HPO_MAX_UNITS];
  int n_seen = 0;
  for (int i = 0; i < n; ++i) {
    int ix = -1;
    for (int j = 0; j < n_seen; ++j) {
      if (seen_key[j] == key[i]) {
        ix = j;
        break;
      }
    }
    if (ix < 0) {
      seen_key[n_seen] = key[i];
      ix = n_seen++;
    }
    out[i] = ix;
  }
}

double hpo_seed_floor(int n, const double* power, const double* memory, const int* type_id,
                      const int* node_id, int n_microbatches, double min_mem, int* out_rgs,
                      double* out_z) {
  int seeds[4][HPO_MAX_UNITS];
  for (int i = 0; i < n; ++i) {
    seeds[0][i] = 0;
    seeds[1][i] = i;
  }
  first_occurrence(n, type_id, seeds[2]);
  first_occurrence(n, node_id, seeds[3]);
  double seed_obj = -1, seed_z = 0;
  int seed_ix = -1;
  for (int k = 0; k < 4; ++k) {
    double z = 0;
    const double obj = evaluate_partition(n, power, memory, seeds[k], n_microbatches,
                                          min_mem, &z);
    if (obj > seed_obj) {
      seed_obj = obj;
      seed_z = z;
      seed_ix = k;
    }
  }
  if (seed_ix >= 0) {
    memcpy(out_rgs, seeds[seed_ix], sizeof(int) * (size_t)n);
    *out_z = seed_z;
  }
  return seed_obj;
}

int hpo_solve_grouping(int n, const double* power, const double* memory,
                       const int* type_id, const int* node_id, int n_microbatches,
                       double min_mem, int exact_threshold, long long node_budget,
                       int top_k, int* out_count, int* out_rgs, double* out_obj,
                       double* out_z, int* out_optimal, hpo_grouping_stats* stats) {
  if (n_microbatches < 1) return 6;           /* :270-272 */
  if (n < 1 || n > HPO_MAX_UNITS) return 6;   /* :274 */
  double total_mem = 0;                       /* :276-277 */
  for (int i = 0; i < n; ++i) total_mem += memory[i];
  if (total_mem < min_mem) return 3;          /* :283-289 */

  search* s = (search*)calloc(1, sizeof(search));
  if (!s) return 5;
  s->n = n;
  s->power = power;
  s->memory = memory;
  s->k_total = n_microbatches;
  s->min_mem = min_mem;
  s->top_k = top_k > 1 ? top_k : 1;                                  /* :295 */
  s->budget = n <= exact_threshold ? -1 : node_budget;               /* :296-297 */
  s->best = (cand*)calloc((size_t)s->top_k + 1, sizeof(cand));

  /* seeds, :206-225 and :299-312; strict '>' keeps the first seed on ties */
  int seeds[4][HPO_MAX_UNITS];
  for (int i = 0; i < n; ++i) {
    seeds[0][i] = 0;
    seeds[1][i] = i;
  }
  first_occurrence(n, type_id, seeds[2]);
  first_occurrence(n, node_id, seeds[3]);
  double seed_obj = -1, seed_z = 0;
  int seed_ix = -1;
  for (int k = 0; k < 4; ++k) {
    double z = 0;
    const double obj = evaluate_partition(n, power, memory, seeds[k], n_microbatches,
                                          min_mem, &z);
    if (obj > seed_obj) {
      seed_obj = obj;
      seed_z = z;
      seed_ix = k;
    }
  }
  s->prune_floor = seed_obj;

  dfs(s, 0);

  const int optimal = !s->aborted;
  int rc = 0;
  if (s->n_best == 0) { /* :318-325 */
    if (seed_obj < 0) {
      rc = 3;
    } else {
      *out_count = 1;
      memcpy(out_rgs, seeds[seed_ix], sizeof(int) * (size_t)n);
      out_obj[0] = seed_obj;
      out_z[0] = seed_z;
      *out_optimal = 0;
    }
  } else if (!optimal && seed_obj > s->best[0].objective) { /* :327-330 */
    *out_count = 1;
    memcpy(out_rgs, seeds[seed_ix], sizeof(int) * (size_t)n);
    out_obj[0] = seed_obj;
    out_z[0] = seed_z;
    *out_optimal = 0;
  } else { /* :331-333 */
    *out_count = s->n_best;
    for (int k = 0; k < s->n_best; ++k) {
      memcpy(out_rgs + (size_t)k * n, s->best[k].rgs, sizeof(int) * (size_t)n);
      out_obj[k] = s->best[k].objective;
      out_z[k] = s->best[k].z;
    }
    *out_optimal = optimal;
  }
  if (stats) *stats = s->st;
  free(s->best);
  free(s);
  return rc;
}

/* --------------------------------------------------------------- partition */

double hpo_stage_time(const double* prof_row, int n_bits, int layers) {
  double total = 0; /* P/src/profile.cpp:180-190 */
  for (int bit = 0; bit < n_bits && (1 << bit) <= layers; ++bit) {
    if (layers & (1 << bit)) total += prof_row[bit];
  }
  return total;
}

double hpo_stage_memory(int layers, int stage_index, int total_stages, int tp, double ppb,
                        double pab, double opt_mult, int k_total) {
  if (layers == 0) return 0; /* P/src/profile.cpp:226-232 */
  const double fixed = (double)layers * ppb * (1.0 + opt_mult) / (double)tp; /* :200-203 */
  const int in_flight = k_total < total_stages - stage_index + 1
                            ? k_total
                            : total_stages - stage_index + 1; /* :205-215 */
  const double variable = (double)layers * pab * (double)in_flight / (double)tp;
  return fixed + variable;
}

/* first missing bit of a profile row for `layers`, or -1 */
static int missing_bit(const double* prof_row, int n_bits, int layers) {
  for (int bit = 0; (1 << bit) <= layers; ++bit) {
    if (layers & (1 << bit)) {
      if (bit >= n_bits || !(prof_row[bit] > 0)) return bit;
    }
  }
  return -1;
}

int hpo_balance_workload(int n_layers, int P, int n_bits, const double* prof,
                         const double* mem_capacity, const int* stage_index, int tp,
                         double ppb, double pab, double opt_mult, int k_total,
                         int allow_zero, int* out_layers, double* out_times,
                         double* out_bottleneck, int* missing_stage, int* missing_layers) {
  const int n = n_layers;
  if (P == 0) return 6;                         /* P/src/partition.cpp:53 */
  const int min_layers = allow_zero ? 0 : 1;    /* :54 */
  if (n < min_layers * P) return 3;             /* :55-58 */
  const size_t W = (size_t)n + 1;
  double* eval = (double*)malloc(sizeof(double) * W * (size_t)P);
  double* best = (double*)malloc(sizeof(double) * W * ((size_t)P + 1));
  for (int i = 0; i < P; ++i) { /* :60-70 */
    double* row = eval + (size_t)i * W;
    for (int l = 0; l <= n; ++l) row[l] = INFINITY;
    for (int l = min_layers; l <= n; ++l) {
      const double bytes = hpo_stage_memory(l, stage_index[i], P, tp, ppb, pab, opt_mult,
                                            k_total);
      if (bytes <= mem_capacity[i]) {
        if (l == 0) {
          row[l] = 0;
        } else {
          const int mb = missing_bit(prof + (size_t)i * n_bits, n_bits, l);
          if (mb >= 0) {
            *missing_stage = i;
            *missing_layers = 1 << mb;
            free(eval);
            free(best);
            return 6;
          }
          row[l] = hpo_stage_time(prof + (size_t)i * n_bits, n_bits, l);
        }
      }
    }
    if (allow_zero) row[0] = 0;
  }
  for (size_t k = 0; k < W * ((size_t)P + 1); ++k) best[k] = INFINITY; /* :72-83 */
  best[(size_t)P * W + 0] = 0;
  for (int i = P - 1; i >= 0; --i) {
    for (int r = 0; r <= n; ++r) {
      double b = INFINITY;
      for (int l = min_layers; l <= r; ++l) {
        const double e = eval[(size_t)i * W + l];
        const double nb = best[(size_t)(i + 1) * W + (r - l)];
        if (e == INFINITY || nb == INFINITY) continue;
        const double m = e < nb ? nb : e; /* std::max */
        b = m < b ? m : b;                /* std::min */
      }
      best[(size_t)i * W + r] = b;
    }
  }
  const double bottleneck = best[n];
  if (bottleneck == INFINITY) { /* :85-89 */
    free(eval);
    free(best);
    return 3;
  }
  int remaining = n; /* :91-106 */
  double bn = 0;
  for (int i = 0; i < P; ++i) {
    int chosen = -1;
    for (int l = remaining; l >= min_layers; --l) {
      if (eval[(size_t)i * W + l] <= bottleneck &&
          best[(size_t)(i + 1) * W + (remaining - l)] <= bottleneck) {
        chosen = l;
        break;
      }
    }
    if (chosen < 0) {
      free(eval);
      free(best);
      return 5;
    }
    out_layers[i] = chosen;
    out_times[i] = eval[(size_t)i * W + chosen];
    bn = (i == 0 || out_times[i] > bn) ? out_times[i] : bn;
    remaining -= chosen;
  }
  *out_bottleneck = bn; /* :108 */
  free(eval);
  free(best);
  return remaining == 0 ? 0 : 5;
}

/* -------------------------------------------------------------------- cost */

void hpo_estimate_iteration(int G, const int* group_off, const int* microbatches,
                            const int* stage_layers, const double* stage_time,
                            const int* stage_node, const int* stage_rank0, int n_layers,
                            int tp, double ppb, double pab, double intra_bw,
                            double inter_bw, int sync_max, double* out_fill,
                            double* out_steady, double* out_total, double* out_bubble,
                            double* out_t_sync, double* out_t_star) {
  double worst = 0; /* P/src/cost.cpp:122-147 */
  for (int g = 0; g < G; ++g) {
    const int s0 = group_off[g], P = group_off[g + 1] - group_off[g];
    double fill = 0, peak = 0;
    for (int i = 0; i < P; ++i) {
      /* stage_times_with_comm, :43-69; boundary_seconds :29-39 (rank-matched
       * devices of a TP unit share its node, so the min link is intra iff the
       * two units share a node; P/src/cluster.cpp:187-192) */
      double t = stage_time[s0 + i];
      if (i + 1 < P) {
        const double bw = stage_node[s0 + i] == stage_node[s0 + i + 1] ? intra_bw : inter_bw;
        t += pab / bw;
      }
      if (i > 0) {
        const double bw = stage_node[s0 + i - 1] == stage_node[s0 + i] ? intra_bw : inter_bw;
        t += pab / bw;
      }
      fill += t;
      peak = t > peak ? t : peak;
    }
    const int K = microbatches[g];
    out_fill[g] = fill;
    out_steady[g] = (double)(K - 1) * peak;
    out_total[g] = out_fill[g] + out_steady[g];
    out_bubble[g] = (double)(P - 1) / (double)(K + P - 1);
    worst = out_total[g] > worst ? out_total[g] : worst;
  }
  /* estimate_sync, :73-120 */
  double total = 0;
  int* hold_rank = (int*)malloc(sizeof(int) * (size_t)(G > 0 ? G : 1));
  int* hold_node = (int*)malloc(sizeof(int) * (size_t)(G > 0 ? G : 1));
  for (int layer = 0; layer < n_layers; ++layer) {
    int d = 0;
    for (int g = 0; g < G; ++g) {
      int begin = 0;
      for (int s = group_off[g]; s < group_off[g + 1]; ++s) {
        const int end = begin + stage_layers[s];
        if (layer >= begin && layer < end) {
          hold_rank[d] = stage_rank0[s];
          hold_node[d] = stage_node[s];
          ++d;
          break;
        }
        begin = end;
      }
    }
    double seconds = 0;
    if (d >= 2) {
      for (int a = 1; a < d; ++a) { /* sort by global rank (distinct) */
        for (int b = a; b > 0 && hold_rank[b] < hold_rank[b - 1]; --b) {
          int t = hold_rank[b];
          hold_rank[b] = hold_rank[b - 1];
          hold_rank[b - 1] = t;
          t = hold_node[b];
          hold_node[b] = hold_node[b - 1];
          hold_node[b - 1] = t;
        }
      }
      double min_bw = 0;
      for (int i = 0; i < d; ++i) {
        const double bw = hold_node[i] == hold_node[(i + 1) % d] ? intra_bw : inter_bw;
        min_bw = i == 0 ? bw : (bw < min_bw ? bw : min_bw);
      }
      const double volume = ppb / (double)tp;
      seconds = 2.0 * (double)(d - 1) / (double)d * volume / min_bw;
    }
    total = sync_max ? (seconds > total ? seconds : total) : total + seconds;
  }
  free(hold_rank);
  free(hold_node);
  *out_t_sync = total;
  *out_t_star = worst + total;
}
