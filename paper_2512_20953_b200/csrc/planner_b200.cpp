// planner_b200.cpp — drop-in replacement of the reference planner translation
// unit (P/src/planner.cpp; P = /root/reference/proj): the same
//   hetplan::plan_cluster(spec, cfg, profile, memmodel, PlannerOptions)
// (P/include/hetplan/planner.hpp:43-45), reached from hp_plan_compute
// (P/src/c_api.cpp:185-208) unchanged.
//
// Control flow, status strings and exception behaviour follow planner.cpp
// line by line; the arithmetic of the hot path runs on the B200:
//   * every TP dimension's DP-grouping search is one problem of ONE batched
//     hpk_grouping_search launch (grouping.cpp:269-335 semantics, bit-exact);
//   * every candidate's stage-mapper DP-affinity pass (stage_map.cpp:188-214)
//     is one CTA of ONE batched hpk_stage_affinity launch;
//   * every candidate's layer partition + Eq. (1) cost is one CTA of ONE
//     batched hpk_partition_cost launch (partition.cpp:51-110, cost.cpp:29-147).
// Host work left here, all restated (no reference function is called for any
// SURVEY 8 row): option handling, TP dimensions and TP-unit formation (R1-R2),
// MIN_mem (R3), the stage mapper's joint / fallback placement
// (stage_map.cpp:63-186), plan assembly and validation (R17). There is no CPU
// fallback: without a CUDA device plan_cluster throws InternalError.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <thread>
#include <cmath>
#include <iostream>
#include <map>
#include <numeric>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "hetplan/cost.hpp"
#include "hetplan/grouping.hpp"
#include "hetplan/partition.hpp"
#include "hetplan/planner.hpp"
#include "hetplan/stage_map.hpp"
#include "hetplan/util.hpp"
#include "hetplan_b200.h"


namespace hetplan {

// sim_b200.cpp: every group of every plan through the GPU 1F1B simulator
std::vector<PlanSimResult> simulate_plans(const std::vector<const ParallelPlan*>& plans,
                                          const std::vector<const ProfileTable*>& profiles,
                                          const std::vector<const ModelConfig*>& cfgs,
                                          const std::vector<const ClusterSpec*>& specs,
                                          const SimOptions& options);

namespace {

// ---- R1-R3 and plan validation, restated (no reference code runs for them).

// R1, enumerate_tp_dims (grouping.cpp:341-350): the divisors of the gcd of the
// nodes' GPU counts, ascending; [1] when there is no node.
std::vector<int> valid_tp_dims(const ClusterSpec& spec) {
  int g = 0;
  for (const auto& nd : spec.nodes) g = std::gcd(g, nd.gpu_count);
  std::vector<int> dims;
  for (int t = 1; t <= g; ++t)
    if (g % t == 0) dims.push_back(t);
  if (dims.empty()) dims.push_back(1);
  return dims;
}

// derive_power (profile.cpp:234-262): T_ref / T_type at the largest layer
// count profiled for every type at tp_dim.
std::map<std::string, double> derived_powers(const ProfileTable& table, const std::string& ref,
                                             int tp_dim) {
  const std::vector<std::string> types = table.gpu_types();
  if (std::find(types.begin(), types.end(), ref) == types.end()) {
    throw InvalidArgumentError("derive_power: reference type '" + ref +
                               "' not in profile table");
  }
  std::vector<int> common = table.layer_counts(types.front(), tp_dim);
  for (const auto& t : types) {
    const std::vector<int> counts = table.layer_counts(t, tp_dim);
    std::vector<int> keep;
    for (int c : common)
      if (std::binary_search(counts.begin(), counts.end(), c)) keep.push_back(c);
    common.swap(keep);
  }
  if (common.empty()) {
    throw InvalidArgumentError("derive_power: no layer count profiled for every type at tp=" +
                               std::to_string(tp_dim));
  }
  const int anchor = common.back();
  const double t_ref = table.at(ref, tp_dim, anchor);
  std::map<std::string, double> out;
  for (const auto& t : types) out[t] = t_ref / table.at(t, tp_dim, anchor);
  return out;
}

// One device as the grouping sees it (GroupingDevice, grouping.hpp:38-43).
struct Dev {
  DeviceId id;
  const std::string* type;
  double power, memory;
};

// grouping_devices (planner.cpp:34-50): every device in spec order with its
// type's power (or the derived one) and memory.
std::vector<Dev> device_list(const ClusterSpec& spec,
                             const std::map<std::string, double>* powers) {
  std::vector<Dev> out;
  for (const auto& nd : spec.nodes) {
    for (int r = 0; r < nd.gpu_count; ++r) {
      const DeviceId d{nd.node_id, r};
      const GpuType& t = spec.type_of(d);  // first node with this id (cluster.cpp:57-62)
      double g = t.compute_power;
      if (powers) {
        auto it = powers->find(t.name);
        if (it == powers->end()) {
          throw InvalidArgumentError("derived powers missing GPU type " + t.name);
        }
        g = it->second;
      }
      out.push_back({d, &t.name, g, t.memory});
    }
  }
  return out;
}

// R2, build_tp_units (grouping.cpp:40-75): devices ordered by (node, rank);
// each node's run is cut into consecutive blocks of tp_dim same-type devices;
// power and memory summed in rank order from 0.
std::vector<TpUnit> tp_units(std::vector<Dev> devs, int tp_dim) {
  if (tp_dim < 1) throw InvalidArgumentError("tp_dim must be >= 1");
  std::sort(devs.begin(), devs.end(), [](const Dev& a, const Dev& b) { return a.id < b.id; });
  std::vector<TpUnit> units;
  for (size_t i = 0; i < devs.size();) {
    size_t j = i;
    while (j < devs.size() && devs[j].id.node_id == devs[i].id.node_id) ++j;
    if ((j - i) % (size_t)tp_dim != 0) {
      throw InfeasibleError("tp_dim " + std::to_string(tp_dim) +
                            " does not divide the GPU count of node " +
                            std::to_string(devs[i].id.node_id) + " (divisibility)");
    }
    for (size_t b = i; b < j; b += (size_t)tp_dim) {
      TpUnit u;
      u.node_id = devs[b].id.node_id;
      u.gpu_type = *devs[b].type;
      for (size_t k = b; k < b + (size_t)tp_dim; ++k) {
        if (*devs[k].type != u.gpu_type) {
          throw InfeasibleError("mixed GPU types on node " + std::to_string(u.node_id) +
                                "; TP units must be same-type");
        }
        u.devices.push_back(devs[k].id);
        u.power += devs[k].power;
        u.memory += devs[k].memory;
      }
      units.push_back(std::move(u));
    }
    i = j;
  }
  return units;
}

// R3, MemoryModel::required_group_memory (profile.cpp:217-224): MIN_mem is
// tp-independent, L·ppb·(1+om) + L·pab, unless the model overrides it.
double group_memory_floor(const MemoryModel& mm, const ModelConfig& cfg) {
  if (mm.min_mem_override > 0) return mm.min_mem_override;
  return cfg.n_layers * mm.per_layer_param_bytes * (1.0 + mm.optimizer_multiplier) +
         cfg.n_layers * mm.per_layer_activation_bytes;
}

// ParallelPlan::validate (plan.cpp:30-51): the same invariants in the same
// order, raising InternalError with the reference's text.
void check_plan(const ParallelPlan& plan) {
  auto need = [](bool ok, const char* what, const char* expr) {
    if (!ok) {
      throw InternalError(std::string("invariant violated: ") + what + " [" + expr + "]");
    }
  };
  need(plan.tp_dim >= 1, "tp_dim >= 1", "tp_dim >= 1");
  need(!plan.groups.empty(), "plan has at least one group", "!groups.empty()");
  std::set<DeviceId> seen;
  for (const auto& group : plan.groups) {
    need(!group.stages.empty(), "group has at least one stage", "!group.stages.empty()");
    int expected = 1;
    int cursor = 0;
    for (const auto& st : group.stages) {
      need(st.stage_index == expected++, "stage indices contiguous from 1",
           "st.stage_index == expected_index++");
      need((int)st.devices.size() == plan.tp_dim, "stage holds tp_dim devices",
           "static_cast<int>(st.devices.size()) == tp_dim");
      need(st.layer_begin == cursor, "layer ranges tile [0, n_layers)",
           "st.layer_begin == cursor");
      need(st.layer_end >= st.layer_begin, "layer range is not inverted",
           "st.layer_end >= st.layer_begin");
      cursor = st.layer_end;
      for (const auto& d : st.devices) {
        need(d.node_id == st.devices.front().node_id, "TP unit is co-located",
             "d.node_id == st.devices.front().node_id");
        need(seen.insert(d).second, "device appears exactly once in the plan",
             "seen.insert(d).second");
      }
    }
    need(cursor == plan.n_layers, "every group covers all layers", "cursor == n_layers");
  }
}

// split_microbatches (plan.cpp:53-62): earlier groups take the remainder.
std::vector<int> microbatch_split(int total, int n_groups) {
  HP_CHECK(n_groups >= 1, "at least one group");
  std::vector<int> out(n_groups, 0);
  const int base = total / n_groups;
  const int rem = total % n_groups;
  for (int j = 0; j < n_groups; ++j) out[j] = std::max(1, base + (j < rem ? 1 : 0));
  return out;
}

// Deferred exception, re-thrown where the reference would have thrown it.
struct Pending {
  enum Kind { NONE, INVALID, INFEASIBLE, INTERNAL } kind = NONE;
  std::string msg;
  [[noreturn]] void raise() const {
    if (kind == INVALID) throw InvalidArgumentError(msg);
    if (kind == INFEASIBLE) throw InfeasibleError(msg);
    throw InternalError(msg);
  }
};

template <typename Fn>
Pending capture(Fn&& fn) {
  Pending p;
  try {
    fn();
  } catch (const InvalidArgumentError& e) {
    p.kind = Pending::INVALID;
    p.msg = e.what();
  } catch (const InfeasibleError& e) {
    p.kind = Pending::INFEASIBLE;
    p.msg = e.what();
  } catch (const InternalError& e) {
    p.kind = Pending::INTERNAL;
    p.msg = e.what();
  }
  return p;
}

// Stage mapping, map_nodes_and_stages (stage_map.cpp:63-216), restated: the
// joint weakest-type-first phase and the fallback fill (:76-186) run here on
// the host (cheap, data-dependent control); the DP-affinity hill climb
// (:188-214, ~3.5 ms per 64-unit candidate on the host) runs on the GPU for
// every candidate of the planning call in one hpk_stage_affinity launch.
// Units are pooled in (node, first local rank) order (:84-91) — a strict
// order, so the unstable sort of the reference is deterministic.
StageMapping premap_stages(const ClusterSpec& spec, const GroupingSolution& grouping) {
  for (const auto& kv : grouping.assignment) {
    if (!spec.has_device(kv.first)) {
      throw InvalidArgumentError("grouping references device " + kv.first.str() +
                                 " absent from the cluster spec");
    }
  }
  const int G = (int)grouping.groups.size();
  // dense type ids; need[g][type] = the group's remaining slots of that type
  std::map<std::string, int> tid;
  std::vector<const TpUnit*> pool;
  for (const auto& grp : grouping.groups)
    for (const auto& u : grp) {
      pool.push_back(&u);
      tid.emplace(u.gpu_type, (int)tid.size());
    }
  const int T = (int)tid.size();
  std::vector<int> need((size_t)G * T, 0);
  for (int g = 0; g < G; ++g)
    for (const auto& u : grouping.groups[g]) need[(size_t)g * T + tid.at(u.gpu_type)] += 1;
  std::sort(pool.begin(), pool.end(), [](const TpUnit* a, const TpUnit* b) {
    if (a->node_id != b->node_id) return a->node_id < b->node_id;
    return a->devices.front().local_rank < b->devices.front().local_rank;
  });
  const int N = (int)pool.size();
  std::vector<int> ptype(N);
  for (int i = 0; i < N; ++i) ptype[i] = tid.at(pool[i]->gpu_type);
  std::vector<char> taken(N, 0);
  // types by (power of the first pooled unit of the type, name) (:93-104)
  std::vector<std::pair<double, std::string>> order;
  {
    std::vector<char> seen(T, 0);
    for (int i = 0; i < N; ++i)
      if (!seen[ptype[i]]) {
        seen[ptype[i]] = 1;
        order.push_back({pool[i]->power, pool[i]->gpu_type});
      }
    std::sort(order.begin(), order.end());
  }
  StageMapping mapping;
  mapping.groups.assign(G, {});
  std::vector<int> next_stage(G, 1);
  auto place = [&](int g, int i) {
    taken[i] = 1;
    need[(size_t)g * T + ptype[i]] -= 1;
    mapping.groups[g].stages.push_back({next_stage[g]++, *pool[i]});
  };
  // joint phase (:106-163): the weakest type with units left goes to every
  // group at once, all from the lowest-id node holding >= G of them
  while (true) {
    int t = -1;
    std::string tname;
    for (const auto& pr : order) {
      const int k = tid.at(pr.second);
      for (int i = 0; i < N && t < 0; ++i)
        if (!taken[i] && ptype[i] == k) t = k;
      if (t >= 0) {
        tname = pr.second;
        break;
      }
    }
    if (t < 0) break;
    bool all_need = true;
    for (int g = 0; g < G && all_need; ++g) all_need = need[(size_t)g * T + t] > 0;
    if (!all_need) {
      mapping.joint_phase_completed = false;
      mapping.halt_reason = "type " + tname + " is not needed by every DP group";
      break;
    }
    std::map<int, std::vector<int>> by_node;  // ascending node id, pool order inside
    for (int i = 0; i < N; ++i)
      if (!taken[i] && ptype[i] == t) by_node[pool[i]->node_id].push_back(i);
    const std::vector<int>* supply = nullptr;
    for (const auto& kv : by_node)
      if ((int)kv.second.size() >= G) {
        supply = &kv.second;
        break;
      }
    if (!supply) {
      mapping.joint_phase_completed = false;
      mapping.halt_reason = "no single node can host a " + tname + " stage for every DP group";
      break;
    }
    for (int g = 0; g < G; ++g) place(g, (*supply)[g]);
  }
  // fallback (:165-186): leftovers in (power, node, rank) order, each to the
  // first group still needing its type
  std::vector<int> rest;
  for (int i = 0; i < N; ++i)
    if (!taken[i]) rest.push_back(i);
  std::sort(rest.begin(), rest.end(), [&](int a, int b) {
    const TpUnit& x = *pool[a];
    const TpUnit& y = *pool[b];
    if (x.power != y.power) return x.power < y.power;
    if (x.node_id != y.node_id) return x.node_id < y.node_id;
    return x.devices.front().local_rank < y.devices.front().local_rank;
  });
  for (int i : rest) {
    int g = 0;
    while (g < G && need[(size_t)g * T + ptype[i]] <= 0) ++g;
    HP_CHECK(g < G, "every pooled unit belongs to some group's type multiset");
    place(g, i);
  }
  for (int g = 0; g < G; ++g) {
    HP_CHECK(mapping.groups[g].stages.size() == grouping.groups[g].size(),
             "stage count matches the grouping");
  }
  return mapping;
}

// The GPU affinity pass's inputs for a pre-mapped candidate.
struct AffinityIn {
  std::vector<int> goff, type, node, perm;
};
AffinityIn affinity_inputs(const StageMapping& m) {
  AffinityIn a;
  std::map<std::string, int> tid;
  a.goff.push_back(0);
  for (const auto& g : m.groups) {
    for (const auto& st : g.stages) {
      a.type.push_back(tid.emplace(st.unit.gpu_type, (int)tid.size()).first->second);
      a.node.push_back(st.unit.node_id);
    }
    a.goff.push_back((int)a.type.size());
  }
  a.perm.assign(a.type.size(), 0);
  return a;
}
// Applies the swaps (slot s now holds the unit of slot perm[s]).
void apply_affinity(StageMapping& m, const AffinityIn& a) {
  std::vector<TpUnit> units;
  for (const auto& g : m.groups)
    for (const auto& st : g.stages) units.push_back(st.unit);
  size_t s = 0;
  for (auto& g : m.groups)
    for (auto& st : g.stages) st.unit = units[a.perm[s++]];
}

// One candidate = one grouping of one TP dimension, mapped to stages.
struct Candidate {
  int tp = 0;
  const GroupingSolution* grouping = nullptr;
  Pending map_error;  // from the stage mapping (premap_stages)
  StageMapping mapping;
  AffinityIn aff;     // the GPU affinity pass of the mapping
  std::vector<int> microbatches;
  // flattened GPU inputs
  std::vector<int> goff, stype, sindex, snode, srank0;
  std::vector<double> scap, prof;
  std::vector<std::string> type_rows;
  int n_bits = 0;
  // GPU outputs
  std::vector<int> layers;
  std::vector<double> stime, smem, fill, steady, total, bubble;
  hpk_plan_result res{};
};

struct TpWork {
  int tp = 0;
  CandidateSummary summary;
  bool decided = false;          // summary final before search (divisibility, (3b) total)
  Pending pre;                   // exception the reference raises before/inside the search
  std::vector<TpUnit> units;
  double min_mem = 0;
  int problem = -1;              // index into the GPU search batch
  std::vector<GroupingSolution> groupings;
  std::vector<int> cand_ix;      // into candidates, grouping order
};

[[noreturn]] void gpu_fail(int rc) {
  const char* msg = hpk_last_error();
  std::string m = msg && *msg ? msg : "hetplan_b200: GPU engine failure";
  if (rc == 6) throw InvalidArgumentError(m);
  throw InternalError(m);
}

// One plan_cluster call, split at its two GPU launches so that many calls
// (a replanning sweep) share one grouping-search launch and one
// partition/cost launch (hp_plan_compute_batch).
struct PlanJob {
  const ClusterSpec& spec;
  const ModelConfig& cfg;
  const ProfileTable& profile;
  const MemoryModel& memmodel;
  const PlannerOptions& options;
  std::vector<int> tp_dims, valid;
  std::optional<std::map<std::string, double>> derived;
  std::map<std::string, int> type_key;
  std::vector<TpWork> work;
  std::vector<hpk_grouping_problem> problems;
  std::vector<std::vector<double>> pw, pm;
  std::vector<std::vector<int>> tk, nk;
  std::vector<hpk_grouping_result> gres;
  std::vector<std::vector<int>> rgs_buf;
  std::vector<std::vector<double>> obj_buf, z_buf;
  std::vector<Candidate> cands;
  std::vector<hpk_plan_candidate> pin;
  std::vector<hpk_affinity_problem> pin_aff;  // the affinity pass of each pin entry
  std::vector<int> pin_of;
  std::vector<hpk_plan_result> pres;
  std::exception_ptr error;  // raised by a phase; the job is finished
  std::optional<ParallelPlan> plan;
  PlanJob(const ClusterSpec& s, const ModelConfig& c, const ProfileTable& p, const MemoryModel& m,
          const PlannerOptions& o)
      : spec(s), cfg(c), profile(p), memmodel(m), options(o) {}
};

// planner.cpp:116-133 and phase 1: per-TP prechecks in the reference's order
void job_prepare(PlanJob& J) {
  const ClusterSpec& spec = J.spec;
  const ModelConfig& cfg = J.cfg;
  const ProfileTable& profile = J.profile;
  const MemoryModel& memmodel = J.memmodel;
  const PlannerOptions& options = J.options;
  auto& tp_dims = J.tp_dims;
  auto& valid = J.valid;
  auto& derived = J.derived;
  auto& type_key = J.type_key;
  auto& work = J.work;
  auto& problems = J.problems;
  auto& pw = J.pw;
  auto& pm = J.pm;
  auto& tk = J.tk;
  auto& nk = J.nk;
  // planner.cpp:119-126
  tp_dims = options.tp_dims;
  valid = valid_tp_dims(spec);
  if (tp_dims.empty()) {
    tp_dims = valid;
  } else {
    std::sort(tp_dims.begin(), tp_dims.end());
    tp_dims.erase(std::unique(tp_dims.begin(), tp_dims.end()), tp_dims.end());
  }
  // planner.cpp:128-133
  if (options.derive_power) {
    std::string ref = options.power_reference;
    if (ref.empty()) ref = spec.gpu_types.begin()->first;
    derived = derived_powers(profile, ref, 1);
  }
  for (const auto& [name, t] : spec.gpu_types) {
    (void)t;
    type_key.emplace(name, (int)type_key.size());
  }

  // ---- phase 1: per-TP prechecks in the reference's order (grouping.cpp:270-289)
  work.assign(tp_dims.size(), TpWork{});
  problems.reserve(tp_dims.size());
  for (size_t w = 0; w < tp_dims.size(); ++w) {
    TpWork& tw = work[w];
    const int tp = tp_dims[w];
    tw.tp = tp;
    tw.summary.tp_dim = tp;
    if (std::find(valid.begin(), valid.end(), tp) == valid.end()) {
      tw.summary.status = "infeasible: tp_dim does not divide every node's GPU count "
                          "(divisibility)";
      tw.decided = true;
      continue;
    }
    std::vector<Dev> devices;
    tw.pre = capture([&] {
      devices = device_list(spec, derived ? &*derived : nullptr);
      tw.min_mem = options.min_mem_override > 0 ? options.min_mem_override
                                                : group_memory_floor(memmodel, cfg);
      double total_dev = 0;
      for (const auto& d : devices) total_dev += d.memory;
      const double big_l = std::max(total_dev, tw.min_mem) * 2 + 1;
      if (cfg.n_microbatches < 1) {
        throw InvalidArgumentError("grouping: n_microbatches must be >= 1");
      }
      tw.units = tp_units(devices, tp);
      if (tw.units.empty()) throw InvalidArgumentError("grouping: no devices");
      double total_mem = 0;
      for (const auto& u : tw.units) total_mem += u.memory;
      if (big_l > 0 && big_l <= tw.min_mem) {
        throw InvalidArgumentError("grouping: big_l must exceed min_mem");
      }
      if (total_mem < tw.min_mem) {
        throw InfeasibleError("grouping infeasible: total memory " + format_double(total_mem) +
                              " B < MIN_mem " + format_double(tw.min_mem) +
                              " B; no DP group assignment can satisfy the group memory "
                              "constraint (3b)");
      }
    });
    if (tw.pre.kind == Pending::INFEASIBLE) {
      tw.summary.status = std::string("infeasible: ") + tw.pre.msg;
      tw.pre = Pending{};
      tw.decided = true;
      continue;
    }
    if (tw.pre.kind != Pending::NONE) continue;  // raised when this TP is reached
    const int n = (int)tw.units.size();
    pw.emplace_back(n);
    pm.emplace_back(n);
    tk.emplace_back(n);
    nk.emplace_back(n);
    for (int i = 0; i < n; ++i) {
      pw.back()[i] = tw.units[i].power;
      pm.back()[i] = tw.units[i].memory;
      tk.back()[i] = type_key.at(tw.units[i].gpu_type);
      nk.back()[i] = tw.units[i].node_id;
    }
    hpk_grouping_problem pr;
    pr.n = n;
    pr.n_microbatches = cfg.n_microbatches;
    pr.min_mem = tw.min_mem;
    pr.exact_threshold = options.exact_threshold;
    pr.node_budget = options.node_budget;
    pr.top_k = std::max(1, options.top_k);
    tw.problem = (int)problems.size();
    problems.push_back(pr);
  }
  for (size_t k = 0; k < problems.size(); ++k) {
    problems[k].power = pw[k].data();
    problems[k].memory = pm[k].data();
    problems[k].type_key = tk[k].data();
    problems[k].node_key = nk[k].data();
  }

  J.gres.assign(problems.size(), hpk_grouping_result{});
  J.rgs_buf.assign(problems.size(), {});
  J.obj_buf.assign(problems.size(), {});
  J.z_buf.assign(problems.size(), {});
  for (size_t k = 0; k < problems.size(); ++k) {
    J.rgs_buf[k].assign((size_t)problems[k].top_k * problems[k].n, 0);
    J.obj_buf[k].assign((size_t)problems[k].top_k, 0.0);
    J.z_buf[k].assign((size_t)problems[k].top_k, 0.0);
    J.gres[k].rgs = J.rgs_buf[k].data();
    J.gres[k].objective = J.obj_buf[k].data();
    J.gres[k].z = J.z_buf[k].data();
  }
}

// phase 3: groupings -> stage mapping -> candidate inputs (host)
void job_candidates(PlanJob& J) {
  const ClusterSpec& spec = J.spec;
  auto& work = J.work;
  auto& gres = J.gres;
  auto& cands = J.cands;
  for (auto& tw : work) {
    if (tw.problem < 0) continue;
    const hpk_grouping_result& r = gres[tw.problem];
    if (r.status == 3) {
      tw.summary.status = "infeasible: grouping infeasible: no partition satisfies the group "
                          "memory constraint (3b)";
      tw.decided = true;
      continue;
    }
    const int n = (int)tw.units.size();
    for (int k = 0; k < r.count; ++k) {  // make_solution, grouping.cpp:249-265
      GroupingSolution sol;
      const int* rgs = r.rgs + (size_t)k * n;
      const int m = *std::max_element(rgs, rgs + n) + 1;
      sol.groups.assign(m, {});
      for (int i = 0; i < n; ++i) {
        sol.groups[rgs[i]].push_back(tw.units[i]);
        for (const auto& d : tw.units[i].devices) sol.assignment[d] = rgs[i];
      }
      for (int gi = 0; gi < m; ++gi) sol.valid_groups.push_back(gi);
      sol.z = r.z[k];
      sol.objective = r.objective[k];
      sol.optimal = r.optimal != 0;
      sol.nodes_visited = r.visited;
      tw.groupings.push_back(std::move(sol));
    }
  }
  for (auto& tw : work) {
    for (size_t k = 0; k < tw.groupings.size(); ++k) {
      Candidate c;
      c.tp = tw.tp;
      c.grouping = &tw.groupings[k];
      tw.cand_ix.push_back((int)cands.size());
      cands.push_back(std::move(c));
    }
  }
  // stage mapping, joint + fallback phases (host); the affinity pass follows
  // on the GPU for every candidate of the call (plan_jobs)
  for (auto& c : cands) {
    c.map_error = capture([&] { c.mapping = premap_stages(spec, *c.grouping); });
    if (c.map_error.kind == Pending::NONE) c.aff = affinity_inputs(c.mapping);
  }
}

// phase 3b: mapped candidates -> partition / cost inputs (host)
void job_partition_inputs(PlanJob& J) {
  const ClusterSpec& spec = J.spec;
  const ModelConfig& cfg = J.cfg;
  const ProfileTable& profile = J.profile;
  const MemoryModel& memmodel = J.memmodel;
  const PlannerOptions& options = J.options;
  auto& cands = J.cands;
  auto& pin = J.pin;
  auto& pin_of = J.pin_of;
  auto& pres = J.pres;
  // inputs from the pre-affinity mapping: the fused launch runs the affinity
  // pass and permutes stage_node / stage_rank0 itself (same-type swaps leave
  // types, stage indices and capacities unchanged)
  int n_bits = 0;
  while ((1 << n_bits) <= cfg.n_layers) ++n_bits;
  pin_of.assign(cands.size(), -1);
  for (size_t ci = 0; ci < cands.size(); ++ci) {
    Candidate& c = cands[ci];
    if (c.map_error.kind != Pending::NONE) continue;
    const int G = (int)c.mapping.groups.size();
    c.microbatches = microbatch_split(cfg.n_microbatches, G);
    std::map<std::string, int> row;
    c.goff.push_back(0);
    for (int j = 0; j < G; ++j) {
      for (const auto& slot : c.mapping.groups[j].stages) {
        auto it = row.find(slot.unit.gpu_type);
        if (it == row.end()) {
          it = row.emplace(slot.unit.gpu_type, (int)c.type_rows.size()).first;
          c.type_rows.push_back(slot.unit.gpu_type);
        }
        c.stype.push_back(it->second);
        c.sindex.push_back(slot.stage_index);
        c.scap.push_back(spec.gpu_types.at(slot.unit.gpu_type).memory);
        c.snode.push_back(slot.unit.node_id);
        c.srank0.push_back(spec.global_rank(slot.unit.devices.front()));
      }
      c.goff.push_back((int)c.stype.size());
    }
    c.n_bits = n_bits;
    for (const auto& t : c.type_rows) {
      for (int b = 0; b < n_bits; ++b) {
        c.prof.push_back(profile.has(t, c.tp, 1 << b) ? profile.at(t, c.tp, 1 << b) : 0.0);
      }
    }
    const size_t S = c.stype.size();
    c.layers.assign(S, 0);
    c.stime.assign(S, 0);
    c.smem.assign(S, 0);
    c.fill.assign(G, 0);
    c.steady.assign(G, 0);
    c.total.assign(G, 0);
    c.bubble.assign(G, 0);
    hpk_plan_candidate p;
    p.n_layers = cfg.n_layers;
    p.tp = c.tp;
    p.k_total = cfg.n_microbatches;
    p.n_groups = G;
    p.ppb = memmodel.per_layer_param_bytes;
    p.pab = memmodel.per_layer_activation_bytes;
    p.opt_mult = memmodel.optimizer_multiplier;
    p.cost_ppb = cfg.per_layer_param_bytes;
    p.cost_pab = cfg.per_layer_activation_bytes;
    p.intra_bw = spec.intra_node_bw;
    p.inter_bw = spec.inter_node_bw;
    p.sync_max = options.sync_overlap == SyncOverlap::max ? 1 : 0;
    p.allow_zero = options.allow_zero_layer_stages ? 1 : 0;
    p.group_stage_off = c.goff.data();
    p.microbatches = c.microbatches.data();
    p.stage_type = c.stype.data();
    p.stage_index = c.sindex.data();
    p.stage_mem_capacity = c.scap.data();
    p.stage_node = c.snode.data();
    p.stage_rank0 = c.srank0.data();
    p.n_types = (int)c.type_rows.size();
    p.n_bits = n_bits;
    p.prof = c.prof.data();
    pin_of[ci] = (int)pin.size();
    pin.push_back(p);
    hpk_affinity_problem a;
    a.n_groups = (int)c.aff.goff.size() - 1;
    a.n_slots = (int)c.aff.type.size();
    a.group_off = c.aff.goff.data();
    a.slot_type = c.aff.type.data();
    a.slot_node = c.aff.node.data();
    a.slot_perm = c.aff.perm.data();
    a.swaps = 0;
    J.pin_aff.push_back(a);
  }
  // result buffers of the batched partition + cost launch (phase 4)
  pres.assign(pin.size(), hpk_plan_result{});
  for (size_t ci = 0; ci < cands.size(); ++ci) {
    if (pin_of[ci] < 0) continue;
    Candidate& c = cands[ci];
    hpk_plan_result& r = pres[pin_of[ci]];
    r.stage_layers = c.layers.data();
    r.stage_time = c.stime.data();
    r.stage_mem = c.smem.data();
    r.group_fill = c.fill.data();
    r.group_steady = c.steady.data();
    r.group_total = c.total.data();
    r.group_bubble = c.bubble.data();
  }
}

// phase 5: the reference's selection loop (planner.cpp:138-205), replayed
ParallelPlan job_select(PlanJob& J) {
  const ClusterSpec& spec = J.spec;
  const ModelConfig& cfg = J.cfg;
  const PlannerOptions& options = J.options;
  auto& work = J.work;
  auto& cands = J.cands;
  auto& pres = J.pres;
  auto& pin_of = J.pin_of;
  std::optional<ParallelPlan> best;
  std::vector<CandidateSummary> summaries;
  for (auto& tw : work) {
    if (tw.pre.kind != Pending::NONE) tw.pre.raise();
    if (tw.decided) {
      summaries.push_back(tw.summary);
      continue;
    }
    CandidateSummary summary = tw.summary;
    bool produced = false;
    std::string last_error;
    for (int ci : tw.cand_ix) {
      Candidate& c = cands[ci];
      if (c.map_error.kind != Pending::NONE) {
        if (c.map_error.kind == Pending::INFEASIBLE) {
          last_error = c.map_error.msg;
          continue;
        }
        c.map_error.raise();
      }
      const hpk_plan_result& r = pres[pin_of[ci]];
      const int G = (int)c.mapping.groups.size();
      if (r.status == 3) {  // balance_workload InfeasibleError (partition.cpp:55-58, 85-89)
        const int j = r.fail_group;
        const int P = c.goff[j + 1] - c.goff[j];
        if (r.fail_kind == 1) {
          last_error = "balance_workload: " + std::to_string(cfg.n_layers) + " layers over " +
                       std::to_string(P) + " stages; every stage needs at least one";
        } else {
          last_error =
              "balance_workload: no layer split fits every stage's memory capacity (the "
              "per-stage memory constraint is binding)";
        }
        continue;
      }
      if (r.status == 6) {  // ProfileTable::at / estimate_stage_time (profile.cpp:95-103,181)
        if (r.missing_layers <= 0) {
          throw InvalidArgumentError("estimate_stage_time: n_layers must be >= 1");
        }
        throw InvalidArgumentError("profile table: no entry for " +
                                   c.type_rows[c.stype[r.missing_stage]] +
                                   " tp=" + std::to_string(c.tp) +
                                   " layers=" + std::to_string(r.missing_layers));
      }
      // assemble (planner.cpp:54-112)
      ParallelPlan plan;
      plan.tp_dim = c.tp;
      plan.n_layers = cfg.n_layers;
      plan.n_microbatches_total = cfg.n_microbatches;
      plan.grouping.objective = c.grouping->objective;
      plan.grouping.z = c.grouping->z;
      plan.grouping.optimal = c.grouping->optimal;
      plan.sync_overlap = options.sync_overlap == SyncOverlap::sum ? "sum" : "max";
      int s = 0;
      for (int j = 0; j < G; ++j) {
        const auto& stages = c.mapping.groups[j].stages;
        GroupPlan group;
        group.microbatches = c.microbatches[j];
        int cursor = 0;
        for (const auto& slot : stages) {
          StagePlan st;
          st.stage_index = slot.stage_index;
          st.gpu_type = slot.unit.gpu_type;
          st.devices = slot.unit.devices;
          st.layer_begin = cursor;
          st.layer_end = cursor + c.layers[s];
          cursor = st.layer_end;
          st.est_time_s = c.stime[s];
          st.est_mem_bytes = c.smem[s];
          st.mem_capacity_bytes = spec.gpu_types.at(st.gpu_type).memory;
          group.stages.push_back(std::move(st));
          ++s;
        }
        plan.groups.push_back(std::move(group));
        GroupCost gc;
        gc.microbatches = c.microbatches[j];
        gc.pipeline_fill = c.fill[j];
        gc.steady = c.steady[j];
        gc.total = c.total[j];
        gc.bubble_ratio = c.bubble[j];
        plan.cost.per_group.push_back(gc);
      }
      plan.cost.t_sync = r.t_sync;
      plan.cost.t_star = r.t_star;
      check_plan(plan);
      summary.grouping_objective = c.grouping->objective;
      summary.t_star = plan.cost.t_star;
      summary.status = "candidate";
      produced = true;
      if (!best || plan.cost.t_star < best->cost.t_star) best = std::move(plan);
      break;  // groupings are ordered best-first; take the first that maps
    }
    if (!produced) summary.status = "infeasible: " + last_error;
    summaries.push_back(summary);
  }

  if (!best) {  // planner.cpp:193-200
    std::ostringstream os;
    os << "no feasible plan; per-TP-dimension binding constraints:";
    for (const auto& s : summaries) os << "\n  tp=" << s.tp_dim << ": " << s.status;
    throw InfeasibleError(os.str());
  }
  for (auto& s : summaries) {
    if (s.status == "candidate" && s.tp_dim == best->tp_dim) s.status = "selected";
  }
  best->candidates = summaries;
  // validate_with_sim (planner.cpp:207-219) follows in plan_jobs: every job's
  // selected plan is simulated in one GPU launch (sim_b200.cpp)
  return *best;
}

// planner.cpp:207-219 for every job that asked for it: one simulator launch
// (combined_time, like the reference), then the reference's warnings per job.
void validate_jobs_with_sim(std::vector<PlanJob*>& jobs) {
  std::vector<PlanJob*> sel;
  std::vector<const ParallelPlan*> plans;
  std::vector<const ProfileTable*> profiles;
  std::vector<const ModelConfig*> cfgs;
  std::vector<const ClusterSpec*> specs;
  for (PlanJob* J : jobs) {
    if (J->error || !J->plan || !J->options.validate_with_sim) continue;
    sel.push_back(J);
    plans.push_back(&*J->plan);
    profiles.push_back(&J->profile);
    cfgs.push_back(&J->cfg);
    specs.push_back(&J->spec);
  }
  if (sel.empty()) return;
  SimOptions sim_opts;
  sim_opts.combined_time = true;
  std::vector<PlanSimResult> sims;
  try {
    sims = simulate_plans(plans, profiles, cfgs, specs, sim_opts);
  } catch (...) {
    // the reference raises from inside plan_cluster: the job fails
    for (PlanJob* J : sel) {
      J->plan.reset();
      J->error = std::current_exception();
    }
    return;
  }
  for (size_t k = 0; k < sel.size(); ++k) {
    const ParallelPlan& best = *sel[k]->plan;
    const PlanSimResult& sim = sims[k];
    for (size_t j = 0; j < sim.groups.size(); ++j) {
      const double estimated = best.cost.per_group[j].total;
      const double simulated = sim.groups[j].pipeline.makespan;
      if (estimated > 0 && std::abs(simulated - estimated) / estimated > 0.01) {
        std::cerr << "warning: group " << j << " simulated makespan " << simulated
                  << "s diverges >1% from estimate " << estimated << "s\n";
      }
    }
  }
}

// Runs fn(job) for every unfinished job on up to `threads` host threads; an
// exception finishes that job.
template <typename Fn>
void for_jobs(std::vector<PlanJob*>& jobs, int threads, Fn&& fn) {
  std::atomic<size_t> next{0};
  auto worker = [&] {
    for (size_t i = next++; i < jobs.size(); i = next++) {
      PlanJob& J = *jobs[i];
      if (J.error || J.plan) continue;
      try {
        fn(J);
      } catch (...) {
        J.error = std::current_exception();
      }
    }
  };
  threads = std::max(1, std::min<int>(threads, (int)jobs.size()));
  if (threads == 1) {
    worker();
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
}

// All jobs through the four phases with ONE grouping-search launch and ONE
// partition/cost launch. A GPU failure fails every job that needed the GPU.
// HPK_HOST_TRACE=1: per-phase wall times of plan_jobs on stderr (diagnostics).
struct PhaseClock {
  static constexpr bool on = HPK_HOST_TRACE != 0;  // build-time: -DHPK_HOST_TRACE=1
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  std::ostringstream os;
  void lap(const char* name) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    os << name << " " << std::chrono::duration<double, std::milli>(now - t).count() << " ms  ";
    t = now;
  }
  ~PhaseClock() {
    if (on) std::cerr << "[hpk-host] " << os.str() << "\n";
  }
};

// A failed GPU launch ends the call: every job not finished yet (including
// jobs with no work in that launch) reports the launch's error.
void fail_unfinished(std::vector<PlanJob*>& jobs, const std::exception_ptr& e) {
  for (PlanJob* J : jobs)
    if (!J->error && !J->plan) J->error = e;
}

void plan_jobs(std::vector<PlanJob*>& jobs, int threads) {
  hpk_reset_timing();
  PhaseClock clk;
  for_jobs(jobs, threads, job_prepare);
  clk.lap("prepare");
  // ---- phase 2: one batched GPU search over every TP dimension of every job
  std::vector<hpk_grouping_problem> problems;
  std::vector<std::pair<PlanJob*, size_t>> owner;
  for (PlanJob* J : jobs) {
    if (J->error) continue;
    for (size_t k = 0; k < J->problems.size(); ++k) {
      problems.push_back(J->problems[k]);
      owner.emplace_back(J, k);
    }
  }
  if (!problems.empty()) {
    std::vector<hpk_grouping_result> gres(problems.size());
    for (size_t i = 0; i < problems.size(); ++i) gres[i] = owner[i].first->gres[owner[i].second];
    try {
      if (hpk_device_count() <= 0) {
        throw InternalError("hetplan_b200: no CUDA device visible; the B200 planner has no CPU "
                            "fallback");
      }
      // the plan needs the winners, not the visit counts: exhaustive top-1
      // searches take the enumeration engine
      hpk_search_config scfg;
      hpk_search_config_init(&scfg);
      scfg.enumerate = 1;
      // every visible GPU: the TP-dimension searches of a plan (and the
      // snapshots of a sweep) go longest-first to the least-loaded device
      scfg.device = HPK_ALL_DEVICES;
      const int rc = hpk_grouping_search(problems.data(), (int)problems.size(), gres.data(),
                                         &scfg);
      if (rc != 0) gpu_fail(rc);
    } catch (...) {
      fail_unfinished(jobs, std::current_exception());
      return;
    }
    for (size_t i = 0; i < problems.size(); ++i) owner[i].first->gres[owner[i].second] = gres[i];
  }
  clk.lap("search");
  for_jobs(jobs, threads, job_candidates);
  clk.lap("candidates(premap)");
  for_jobs(jobs, threads, job_partition_inputs);
  clk.lap("partition-inputs");
  // ---- phases 3 + 4 (GPU, one launch): every candidate's stage-mapper affinity
  // pass, then its layer partition + cost
  std::vector<hpk_affinity_problem> aff;
  std::vector<hpk_plan_candidate> pin;
  std::vector<hpk_plan_result> pres;
  std::vector<std::pair<PlanJob*, size_t>> powner;
  for (PlanJob* J : jobs) {
    if (J->error) continue;
    for (size_t k = 0; k < J->pin.size(); ++k) {
      aff.push_back(J->pin_aff[k]);
      pin.push_back(J->pin[k]);
      pres.push_back(J->pres[k]);
      powner.emplace_back(J, k);
    }
  }
  if (!pin.empty()) {
    try {
      const int rc = hpk_affinity_partition_cost(aff.data(), pin.data(), (int)pin.size(),
                                                 pres.data(), -1);
      if (rc != 0) gpu_fail(rc);
    } catch (...) {
      fail_unfinished(jobs, std::current_exception());
      return;
    }
    for (size_t i = 0; i < pin.size(); ++i) powner[i].first->pres[powner[i].second] = pres[i];
  }
  clk.lap("affinity+partition");
  for_jobs(jobs, threads, [](PlanJob& J) {
    for (auto& c : J.cands)
      if (c.map_error.kind == Pending::NONE) apply_affinity(c.mapping, c.aff);
  });
  for_jobs(jobs, threads, [](PlanJob& J) { J.plan = job_select(J); });
  clk.lap("select");
  validate_jobs_with_sim(jobs);
  clk.lap("validate-sim");
}

}  // namespace

ParallelPlan plan_cluster(const ClusterSpec& spec, const ModelConfig& cfg,
                          const ProfileTable& profile, const MemoryModel& memmodel,
                          const PlannerOptions& options) {
  PlanJob job(spec, cfg, profile, memmodel, options);
  std::vector<PlanJob*> jobs{&job};
  plan_jobs(jobs, 1);
  if (job.error) std::rethrow_exception(job.error);
  if (!job.plan) throw InternalError("hetplan_b200: planning ended without a plan");
  return std::move(*job.plan);
}

}  // namespace hetplan

// ------------------------------------------------------------------ batch C ABI
// The reference's opaque handles (P/src/c_api.cpp:35-47), same definitions.
struct hp_cluster {
  hetplan::ClusterSpec spec;
};
struct hp_model {
  hetplan::ModelConfig config;
  hetplan::MemoryModel memory;
};
struct hp_profile {
  hetplan::ProfileTable table;
};
struct hp_plan {
  hetplan::ParallelPlan plan;
};

namespace {
hp_status status_of(const std::exception_ptr& e, std::string* msg) {
  try {
    std::rethrow_exception(e);
  } catch (const hetplan::ParseError& x) {
    *msg = x.what();
    return HP_PARSE_ERROR;
  } catch (const hetplan::InfeasibleError& x) {
    *msg = x.what();
    return HP_INFEASIBLE;
  } catch (const hetplan::UnrecoverableError& x) {
    *msg = x.what();
    return HP_UNRECOVERABLE;
  } catch (const hetplan::InvalidArgumentError& x) {
    *msg = x.what();
    return HP_INVALID_ARGUMENT;
  } catch (const std::exception& x) {
    *msg = x.what();
    return HP_INTERNAL_ERROR;
  } catch (...) {
    *msg = "unknown error";
    return HP_INTERNAL_ERROR;
  }
}
}  // namespace

void hpkp_fail(const std::string& msg);  // hpk_last_error() text (hpk_grouping.cu)

extern "C" int hpk_map_stages(const hp_cluster* cluster, int tp, int n_groupings,
                              const int* rgs, int* out_unit) {
  using namespace hetplan;
  if (!cluster || tp < 1 || n_groupings < 0 || (n_groupings > 0 && (!rgs || !out_unit))) {
    hpkp_fail("hpk_map_stages: bad arguments");
    return -HP_INVALID_ARGUMENT;
  }
  try {
    const ClusterSpec& spec = cluster->spec;
    const std::vector<TpUnit> units = tp_units(device_list(spec, nullptr), tp);
    const int U = (int)units.size();
    std::vector<GroupingSolution> sols(n_groupings);
    std::vector<StageMapping> maps(n_groupings);
    std::vector<AffinityIn> aff(n_groupings);
    std::vector<hpk_affinity_problem> ap(n_groupings);
    for (int g = 0; g < n_groupings; ++g) {
      const int* r = rgs + (size_t)g * U;
      const int m = U ? *std::max_element(r, r + U) + 1 : 0;
      sols[g].groups.assign(m, {});
      for (int u = 0; u < U; ++u) {
        sols[g].groups[r[u]].push_back(units[u]);
        for (const auto& d : units[u].devices) sols[g].assignment[d] = r[u];
      }
      maps[g] = premap_stages(spec, sols[g]);
      aff[g] = affinity_inputs(maps[g]);
      ap[g].n_groups = (int)aff[g].goff.size() - 1;
      ap[g].n_slots = (int)aff[g].type.size();
      ap[g].group_off = aff[g].goff.data();
      ap[g].slot_type = aff[g].type.data();
      ap[g].slot_node = aff[g].node.data();
      ap[g].slot_perm = aff[g].perm.data();
      ap[g].swaps = 0;
    }
    if (n_groupings > 0) {
      const int rc = hpk_stage_affinity(ap.data(), n_groupings, -1);
      if (rc != 0) gpu_fail(rc);
    }
    for (int g = 0; g < n_groupings; ++g) {
      apply_affinity(maps[g], aff[g]);
      int s = 0;
      for (const auto& grp : maps[g].groups)
        for (const auto& slot : grp.stages) {
          int ix = -1;
          for (int u = 0; u < U && ix < 0; ++u)
            if (units[u].devices.front() == slot.unit.devices.front()) ix = u;
          out_unit[(size_t)g * U + s++] = ix;
        }
    }
    return U;
  } catch (...) {
    std::string msg;
    const hp_status st = status_of(std::current_exception(), &msg);
    hpkp_fail(msg);
    return -(int)st;
  }
}

extern "C" hp_status hp_plan_compute_batch(int n, const hp_cluster* const* clusters,
                                           const hp_model* model,
                                           const hp_profile* const* profiles,
                                           const hp_plan_options* options, int host_threads,
                                           hp_plan** out_plans, hp_status* out_status,
                                           char** out_errors) {
  if (n < 0 || (n > 0 && (!clusters || !profiles || !out_plans || !out_status)) || !model) {
    return HP_INVALID_ARGUMENT;
  }
  hetplan::PlannerOptions po;  // as hp_plan_compute (c_api.cpp:191-204)
  if (options) {
    for (int i = 0; i < options->n_tp_dims; ++i) po.tp_dims.push_back(options->tp_dims[i]);
    po.min_mem_override = options->min_mem_override;
    po.exact_threshold = options->exact_threshold;
    po.node_budget = options->node_budget;
    po.top_k = options->top_k;
    po.sync_overlap = options->sync_overlap_max ? hetplan::SyncOverlap::max
                                                : hetplan::SyncOverlap::sum;
    po.validate_with_sim = options->validate_with_sim != 0;
    po.derive_power = options->derive_power != 0;
    if (options->power_reference) po.power_reference = options->power_reference;
  }
  try {
    std::vector<std::unique_ptr<hetplan::PlanJob>> store;
    std::vector<hetplan::PlanJob*> jobs;
    for (int i = 0; i < n; ++i) {
      if (!clusters[i] || !profiles[i]) return HP_INVALID_ARGUMENT;
      store.push_back(std::make_unique<hetplan::PlanJob>(clusters[i]->spec, model->config,
                                                         profiles[i]->table, model->memory, po));
      jobs.push_back(store.back().get());
    }
    int threads = host_threads > 0 ? host_threads : (int)std::thread::hardware_concurrency();
    hetplan::plan_jobs(jobs, std::max(1, threads));
    for (int i = 0; i < n; ++i) {
      out_plans[i] = nullptr;
      std::string msg;
      if (jobs[i]->error) {
        out_status[i] = status_of(jobs[i]->error, &msg);
      } else if (!jobs[i]->plan) {
        out_status[i] = HP_INTERNAL_ERROR;
        msg = "hetplan_b200: planning ended without a plan";
      } else {
        out_status[i] = HP_OK;
        out_plans[i] = new hp_plan{std::move(*jobs[i]->plan)};
      }
      if (out_errors) {
        out_errors[i] = nullptr;
        if (!msg.empty()) {
          out_errors[i] = static_cast<char*>(std::malloc(msg.size() + 1));
          std::memcpy(out_errors[i], msg.c_str(), msg.size() + 1);
        }
      }
    }
  } catch (...) {
    return HP_INTERNAL_ERROR;
  }
  return HP_OK;
}
