// ref_probe.cpp — thin extern "C" probe over the reference library's C++
// internals, linked into oracle/_ref/libhetplan_probe.so together with the
// reference objects compiled from /root/reference/proj/src (see Makefile).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C restatement
// (hetplan_oracle.c) to the reference itself, function by function.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "hetplan/cluster.hpp"
#include "hetplan/grouping.hpp"
#include "hetplan/partition.hpp"
#include "hetplan/pipeline_sim.hpp"
#include "hetplan/profile.hpp"
#include "hetplan/stage_map.hpp"

using namespace hetplan;

extern "C" {

// solve_grouping_topk (P/src/grouping.cpp:269-335) with one device per unit
// (tp_dim = 1): device i lives on node node_id[i] with local rank = its index
// among that node's devices, type "T<type_id>".
// Returns 0 ok, 3 InfeasibleError, 6 InvalidArgumentError, 5 other.
int ref_solve_grouping(int n, const double* power, const double* memory, const int* type_id,
                       const int* node_id, int n_microbatches, double min_mem,
                       int exact_threshold, long long node_budget, int top_k, int* out_count,
                       int* out_rgs, double* out_obj, double* out_z, int* out_optimal,
                       long long* out_visited) {
  try {
    GroupingProblem pb;
    std::vector<int> next_rank(1024, 0);
    for (int i = 0; i < n; ++i) {
      const int node = node_id[i];
      pb.devices.push_back({DeviceId{node, next_rank[node]++},
                            "T" + std::to_string(type_id[i]), power[i], memory[i]});
    }
    pb.tp_dim = 1;
    pb.n_microbatches = n_microbatches;
    pb.min_mem = min_mem;
    pb.big_l = 0;
    pb.exact_threshold = exact_threshold;
    pb.node_budget = node_budget;
    pb.top_k = top_k;
    auto sols = solve_grouping_topk(pb);
    *out_count = static_cast<int>(sols.size());
    for (size_t k = 0; k < sols.size(); ++k) {
      // Unit order in the solver is the DeviceId order; map back to input order.
      std::vector<int> order(n);
      for (int i = 0; i < n; ++i) order[i] = i;
      std::sort(order.begin(), order.end(), [&](int a, int b) {
        return pb.devices[a].id < pb.devices[b].id;
      });
      for (int i = 0; i < n; ++i) {
        out_rgs[k * n + i] = sols[k].assignment.at(pb.devices[i].id);
      }
      out_obj[k] = sols[k].objective;
      out_z[k] = sols[k].z;
      *out_optimal = sols[k].optimal ? 1 : 0;
      *out_visited = sols[k].nodes_visited;
    }
    return 0;
  } catch (const InfeasibleError&) {
    return 3;
  } catch (const InvalidArgumentError&) {
    return 6;
  } catch (...) {
    return 5;
  }
}

// balance_workload (P/src/partition.cpp:51-110) with a profile table built
// from prof[s*n_bits + b] (<= 0: entry absent), one GPU type per stage.
int ref_balance_workload(int n_layers, int P, int n_bits, const double* prof,
                         const double* mem_capacity, const int* stage_index, int tp, double ppb,
                         double pab, double opt_mult, int k_total, int k_group,
                         int allow_zero, int* out_layers, double* out_times,
                         double* out_bottleneck) {
  try {
    ProfileTable table;
    for (int s = 0; s < P; ++s) {
      for (int b = 0; b < n_bits; ++b) {
        if (prof[s * n_bits + b] > 0) {
          table.add("S" + std::to_string(s), tp, 1 << b, prof[s * n_bits + b]);
        }
      }
    }
    ModelConfig cfg;
    cfg.n_layers = n_layers;
    cfg.per_layer_param_bytes = ppb;
    cfg.per_layer_activation_bytes = pab;
    cfg.optimizer_multiplier = opt_mult;
    cfg.n_microbatches = k_total;
    MemoryModel mem = MemoryModel::from_config(cfg);
    PartitionProblem pp;
    pp.n_layers = n_layers;
    pp.n_microbatches = k_group;
    pp.tp_dim = tp;
    pp.profile = &table;
    pp.memmodel = &mem;
    pp.config = &cfg;
    pp.allow_zero_layers = allow_zero != 0;
    for (int s = 0; s < P; ++s) {
      pp.stages.push_back({"S" + std::to_string(s), 1.0, mem_capacity[s], stage_index[s]});
    }
    Partition part = balance_workload(pp);
    for (int s = 0; s < P; ++s) {
      out_layers[s] = part.layers[s];
      out_times[s] = part.stage_times[s];
    }
    *out_bottleneck = part.bottleneck;
    return 0;
  } catch (const InfeasibleError&) {
    return 3;
  } catch (const InvalidArgumentError&) {
    return 6;
  } catch (...) {
    return 5;
  }
}

// map_nodes_and_stages (P/src/stage_map.cpp:63-216) of n_groupings groupings of
// one cluster's TP units: units = build_tp_units over the spec's devices at
// their type powers (planner.cpp:34-50, grouping.cpp:40-75), grouping g puts
// unit u in group rgs[g*U + u]. Writes, per grouping, the unit index held by
// each stage slot (groups in order, stages in order) into out_unit[g*U + s].
// Returns the unit count U (> 0), or -3 / -6 / -5 on Infeasible /
// InvalidArgument / other errors.
int ref_map_stages(const char* cluster_json, int tp, int n_groupings, const int* rgs,
                   int* out_unit) {
  try {
    const ClusterSpec spec = load_cluster_spec(cluster_json);
    std::vector<GroupingDevice> devs;
    for (const auto& d : spec.all_devices()) {
      const GpuType& t = spec.type_of(d);
      devs.push_back({d, t.name, t.compute_power, t.memory});
    }
    const std::vector<TpUnit> units = build_tp_units(devs, tp);
    const int U = static_cast<int>(units.size());
    for (int g = 0; g < n_groupings; ++g) {
      GroupingSolution sol;
      const int* r = rgs + static_cast<size_t>(g) * U;
      int m = 0;
      for (int u = 0; u < U; ++u) m = std::max(m, r[u] + 1);
      sol.groups.assign(m, {});
      for (int u = 0; u < U; ++u) {
        sol.groups[r[u]].push_back(units[u]);
        for (const auto& d : units[u].devices) sol.assignment[d] = r[u];
      }
      const StageMapping mp = map_nodes_and_stages(spec, sol, tp);
      int s = 0;
      for (const auto& grp : mp.groups) {
        for (const auto& slot : grp.stages) {
          int ix = -1;
          for (int u = 0; u < U && ix < 0; ++u)
            if (units[u].devices.front() == slot.unit.devices.front()) ix = u;
          out_unit[static_cast<size_t>(g) * U + s++] = ix;
        }
      }
    }
    return U;
  } catch (const InfeasibleError&) {
    return -3;
  } catch (const InvalidArgumentError&) {
    return -6;
  } catch (...) {
    return -5;
  }
}

// simulate_pipeline (P/src/pipeline_sim.cpp:46-149) on P stages x K
// microbatches: makespan, busy[P], peak[P], and the events in the reference's
// order as (stage, kind 0=F/1=B, microbatch) + (start, end).
// Returns 0 ok, 5 on an invariant failure.
int ref_simulate_pipeline(int P, int K, const double* fwd, const double* bwd, const double* sf,
                          const double* sb, double* makespan, double* busy, int* peak,
                          int* ev_int, double* ev_time) {
  try {
    std::vector<StageTiming> st(P);
    for (int p = 0; p < P; ++p) st[p] = {fwd[p], bwd[p], sf[p], sb[p]};
    const PipelineSimResult r = simulate_pipeline(st, K);
    *makespan = r.makespan;
    for (int p = 0; p < P; ++p) {
      busy[p] = r.busy[p];
      peak[p] = r.peak_in_flight[p];
    }
    for (size_t i = 0; i < r.events.size(); ++i) {
      ev_int[3 * i] = r.events[i].stage;
      ev_int[3 * i + 1] = r.events[i].kind == 'F' ? 0 : 1;
      ev_int[3 * i + 2] = r.events[i].microbatch;
      ev_time[2 * i] = r.events[i].start;
      ev_time[2 * i + 1] = r.events[i].end;
    }
    return 0;
  } catch (...) {
    return 5;
  }
}

}  // extern "C"
