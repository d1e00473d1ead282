// async_emulator.cpp — discrete-event CPU emulation of the asynchronous
// grouping scheduler (design validation harness; NOT product code).
//
// The B200 async engine (hpk_async_kernel) has no waves: warps pull segments
// from a ready set, a running segment is split on demand (the scheduler asks
// the front-most running segments to shed work whenever warps are idle), and a
// scheduler warp per problem commits the ordered segment list continuously.
// This emulator runs that algorithm with the exact serial segment runner of
// wave_emulator.cpp (same node semantics as P/src/grouping.cpp:135-202) in
// simulated time (one time unit = one visit by one warp), so that
//   * exactness (winner, visits, abort flag vs the oracle) is checked on random
//     instances by tests/test_scheduler_emulator.py, and
//   * design choices (ready-set order, split policy, stale-run aborts) can be
//     compared on the real configs before the CUDA kernel is written.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <set>
#include <vector>

namespace {

struct Problem {
  int n;
  std::vector<double> p, m;
  int K;
  double min_mem;
  long long budget;  // < 0 unlimited
  double floor_obj;  // seed objective (prune floor), -1 if none
};

using Path = std::vector<uint8_t>;

struct Best {
  bool has = false;
  double obj = 0;
  int G = 0;
  Path rgs;
};

bool better(double ao, int ag, double bo, int bg) {
  if (ao != bo) return ao > bo;
  return ag < bg;
}

struct RunResult {
  long long visits = 0;
  bool finished = false;
  Path stop;
  Best best;
  double m = -1;
  int a_star = -1;
};

struct GState {
  std::vector<double> gp, gm;
  std::vector<int> gc;
  int G = 0;
};

double eff(const Problem& pb, const GState& s, int g) {
  const int d = s.gc[g];
  const double rho = (double)(d - 1) / (double)(pb.K + d - 1);
  return s.gp[g] * (1.0 - rho);
}

void apply(const Problem& pb, GState& s, int unit, int g) {
  if (g == s.G) {
    s.gp[g] = pb.p[unit];
    s.gm[g] = pb.m[unit];
    s.gc[g] = 1;
    s.G++;
  } else {
    s.gp[g] += pb.p[unit];
    s.gm[g] += pb.m[unit];
    s.gc[g] += 1;
  }
}

void undo(const Problem& pb, GState& s, int unit, int g) {
  if (s.gc[g] == 1 && g == s.G - 1) {
    s.G--;
    s.gc[g] = 0;
  } else {
    s.gp[g] -= pb.p[unit];
    s.gm[g] -= pb.m[unit];
    s.gc[g] -= 1;
  }
}

bool node_passes(const Problem& pb, const GState& s, int next, double cutoff) {
  double bound = 0;
  for (int g = 0; g < s.G; ++g) bound += eff(pb, s, g);
  double rem = 0;
  for (int i = next; i < pb.n; ++i) {
    bound += pb.p[i];
    rem += pb.m[i];
  }
  if (cutoff >= 0 && bound < cutoff) return false;
  double def = 0;
  for (int g = 0; g < s.G; ++g) {
    const double d = pb.min_mem - s.gm[g];
    def += d > 0.0 ? d : 0.0;
  }
  return !(def > rem);
}

int path_cmp(const Path& a, const Path& b) {
  const size_t k = std::min(a.size(), b.size());
  for (size_t i = 0; i < k; ++i)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  if (a.size() == b.size()) return 0;
  return a.size() < b.size() ? -1 : 1;
}

bool is_prefix(const Path& a, const Path& b) {
  if (a.size() > b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i] != b[i]) return false;
  return true;
}

int groups_of(const Path& x, size_t len) {
  int G = 0;
  for (size_t i = 0; i < len; ++i) G = x[i] + 1 > G ? x[i] + 1 : G;
  return G;
}

// Serial segment runner (identical to wave_emulator.cpp): DFS of subtree(u)
// in preorder, at most `cap` visits, stopping before a node >= *end.
RunResult run_segment(const Problem& pb, const Path& u, const Path* end, double cutoff,
                      long long cap) {
  RunResult r;
  GState s;
  s.gp.assign(pb.n + 1, 0);
  s.gm.assign(pb.n + 1, 0);
  s.gc.assign(pb.n + 1, 0);
  for (size_t i = 0; i + 1 < u.size(); ++i) apply(pb, s, (int)i, u[i]);
  Path next = u;
  bool have_next = true;
  double c = cutoff;
  auto advance_from = [&](Path x) -> bool {
    while (true) {
      if (x.size() == u.size()) return false;
      const int d = (int)x.size() - 1;
      const int g = x[d];
      undo(pb, s, d, g);
      if (g + 1 <= s.G) {
        x[d] = (uint8_t)(g + 1);
        next = x;
        return true;
      }
      x.pop_back();
    }
  };
  while (have_next) {
    if (end && path_cmp(next, *end) >= 0) {
      r.finished = true;
      return r;
    }
    if (r.visits >= cap) {
      r.stop = next;
      return r;
    }
    r.visits++;
    const int d = (int)next.size() - 1;
    apply(pb, s, d, next[d]);
    Path x = next;
    if ((int)x.size() == pb.n) {
      bool feas = true;
      double z = 0;
      for (int g = 0; g < s.G; ++g) {
        if (s.gm[g] < pb.min_mem) {
          feas = false;
          break;
        }
        const double e = eff(pb, s, g);
        z = g == 0 ? e : (e < z ? e : z);
      }
      if (feas) {
        const double obj = (double)s.G * z;
        if (!r.best.has || better(obj, s.G, r.best.obj, r.best.G)) {
          r.best.has = true;
          r.best.obj = obj;
          r.best.G = s.G;
          r.best.rgs = x;
        }
        if (obj > r.m) r.m = obj;
        if (obj > c) c = obj;
      }
      have_next = advance_from(x);
      continue;
    }
    if (!node_passes(pb, s, (int)x.size(), c)) {
      if (end && is_prefix(x, *end) && r.a_star < 0) r.a_star = (int)x.size();
      have_next = advance_from(x);
      continue;
    }
    x.push_back(0);
    next = x;
  }
  r.finished = true;
  return r;
}

// ---------------------------------------------------------------- scheduler

enum Status { QUEUED, RUNNING, DONE };

struct Seg {
  Path u;            // root, entered by the segment
  Path end;          // PREFIX end marker (empty: FULL)
  int next = -1;     // ordered list (preorder)
  Status st = QUEUED;
  double pred = -1;  // predicted entering cutoff
  double cut = -1;   // cutoff the run used
  RunResult res;
  bool rerun_exact = false;  // queued by the walker with the exact front cutoff
  // simulation of a running segment
  int warp = -1;
  double t0 = 0, t_end = 0;
  long long cap = 0, horizon = 0;
  bool split_req = false;
  long long gen = 0;  // bumps when the running instance is replaced (stale events)
};

struct Params {
  int warps;
  double pop_cost, split_cost, req_latency, commit_cost;
  int order;         // 0 FIFO ready set, 1 preorder-priority ready set
  int stale_abort;   // 1: a running segment whose cutoff fell behind the front restarts
  long long min_split;  // do not split a run with fewer than this many visits done
  long long slice;      // > 0: a FULL run is preempted after this many units
  long long merge;      // > 0: new pieces become dispatchable only at the scheduler's
                        // next list merge (every `merge` units), like a GPU scheduler
                        // CTA that rebuilds the ordered list periodically
};

struct Event {
  double t;
  int kind;  // 0 finish, 1 split point, 2 scheduler tick
  int seg;
  long long gen;
  bool operator>(const Event& o) const { return t > o.t; }
};

struct Outcome {
  Best best;
  long long visited = 0;
  bool aborted = false;
  double time = 0;
  long long runs = 0, run_visits = 0, splits = 0, reruns = 0, aborts = 0;
};

struct ReadyCmp {
  const std::vector<Seg>* segs;
  int order;
  bool operator()(int a, int b) const {
    const Seg& x = (*segs)[a];
    const Seg& y = (*segs)[b];
    if (x.rerun_exact != y.rerun_exact) return x.rerun_exact;
    if (order == 1) {
      const int c = path_cmp(x.u, y.u);
      if (c != 0) return c < 0;
      if (x.end.empty() != y.end.empty()) return !x.end.empty();
    }
    return a < b;  // FIFO by creation otherwise
  }
};

struct Sim {
  const Problem& pb;
  Params prm;
  std::vector<Seg> segs;
  int head = -1;  // first uncommitted segment of the list
  double C;
  long long V = 0;
  Best gbest;
  bool done = false, aborted = false;
  Path del;       // deletion prefix (ancestor pruned by a PREFIX re-run), empty: none
  bool del_on = false;
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> ev;
  struct ReadyVec {  // the ready set, ordered (preorder or FIFO)
    std::set<int, ReadyCmp>* set;
    void push_back(int s) { set->insert(s); }
    size_t size() const { return set->size(); }
    bool empty() const { return set->empty(); }
  };
  std::set<int, ReadyCmp> ready_set;
  ReadyVec ready;
  std::vector<int> idle;       // idle warps
  double now = 0;
  bool tick_pending = false;
  std::vector<int> pending;  // pieces waiting for the next list merge
  bool merge_pending = false;
  void publish(int id) {
    if (prm.merge <= 0) {
      ready.push_back(id);
      return;
    }
    pending.push_back(id);
    if (!merge_pending) {
      merge_pending = true;
      ev.push({now + (double)prm.merge, 5, 0, 0});
    }
  }
  long long ticks = 0;
  Outcome out;

  Sim(const Problem& p, Params q)
      : pb(p), prm(q), C(p.floor_obj), ready_set(ReadyCmp{&segs, q.order}), ready{&ready_set} {}

  long long remaining_cap() const { return pb.budget < 0 ? (1ll << 60) : pb.budget - V; }

  int pick_ready() {
    if (ready_set.empty()) return -1;
    const int s = *ready_set.begin();
    ready_set.erase(ready_set.begin());
    return s;
  }

  void start(int s, int w, double t) {
    Seg& e = segs[s];
    e.st = RUNNING;
    e.warp = w;
    e.split_req = false;
    e.gen++;
    e.cut = e.rerun_exact ? e.pred : std::max(e.pred, C);
    e.cap = remaining_cap();
    e.t0 = t + prm.pop_cost;
    out.runs++;
    extend(s, std::min<long long>(e.cap, 4096));
    if (prm.slice > 0 && e.end.empty()) ev.push({e.t0 + (double)prm.slice, 4, s, e.gen});
  }

  // The run is computed lazily, doubling its horizon: the result is final
  // once the run finishes or reaches its cap; otherwise re-evaluate later.
  void extend(int s, long long horizon) {
    Seg& e = segs[s];
    e.horizon = horizon;
    e.res = run_segment(pb, e.u, e.end.empty() ? nullptr : &e.end, e.cut, horizon);
    const bool final_ = e.res.finished || horizon >= e.cap;
    e.t_end = e.t0 + (double)(final_ ? e.res.visits : horizon);
    if (final_) {
      out.run_visits += e.res.visits;
      ev.push({e.t_end, 0, s, e.gen});
    } else {
      e.t_end = 1e300;  // still running (for split requests)
      ev.push({e.t0 + (double)horizon, 3, s, e.gen});
    }
  }

  void dispatch(double t) {
    while (!idle.empty()) {
      const int s = pick_ready();
      if (s < 0) break;
      const int w = idle.back();
      idle.pop_back();
      start(s, w, t);
    }
  }

  // Split requests: the front-most running FULL segments shed work while
  // warps are idle and nothing is ready.
  void request_splits(double t) {
    int want = (int)idle.size() - (int)ready.size();
    int scanned = 0;
    for (int s = head; s >= 0 && want > 0 && scanned < 2 * prm.warps + 64; s = segs[s].next, ++scanned) {
      Seg& e = segs[s];
      if (e.st != RUNNING || !e.end.empty() || e.split_req) continue;
      const double tp = t + prm.req_latency;
      if (tp >= e.t_end) continue;
      const long long k = (long long)(tp - e.t0);
      if (k < prm.min_split) continue;
      e.split_req = true;
      ev.push({tp, 1, s, e.gen});
      --want;
    }
  }

  void split(int s, double t, bool keep = true) {
    Seg& e = segs[s];
    const long long k = std::max<long long>(1, (long long)(t - e.t0));
    RunResult r = run_segment(pb, e.u, nullptr, e.cut, k);
    if (r.finished) return;  // nothing left to shed
    out.splits++;
    const double cend = std::max(e.cut, r.m);
    // remainder pieces in preorder: subtree(stop), then right siblings of each
    // ancestor down to u's depth
    std::vector<Path> pieces;
    pieces.push_back(r.stop);
    for (int d = (int)r.stop.size() - 1; d >= (int)e.u.size(); --d) {
      const int Gp = groups_of(r.stop, d);
      for (int c = r.stop[d] + 1; c <= Gp; ++c) {
        Path q(r.stop.begin(), r.stop.begin() + d);
        q.push_back((uint8_t)c);
        pieces.push_back(q);
      }
    }
    // e becomes PREFIX [u, stop), done at t
    out.run_visits += r.visits;
    e.end = r.stop;
    e.res = r;
    e.res.finished = true;
    e.st = DONE;
    e.gen++;
    const int w = e.warp;
    int after = s;
    const int old_next = e.next;
    std::vector<int> ids;
    for (const Path& q : pieces) {
      Seg ns;
      ns.u = q;
      ns.pred = cend;
      segs.push_back(ns);
      ids.push_back((int)segs.size() - 1);
    }
    Seg& e2 = segs[s];  // (vector may have grown)
    for (size_t i = 0; i < ids.size(); ++i) {
      segs[ids[i]].next = i + 1 < ids.size() ? ids[i + 1] : old_next;
      (void)after;
    }
    e2.next = ids[0];
    // the splitting warp keeps the first (deepest) piece, the rest become ready
    if (keep) {
      for (size_t i = 1; i < ids.size(); ++i) publish(ids[i]);
      start(ids[0], w, t + prm.split_cost - prm.pop_cost);
    } else {  // preempted: every piece goes back to the ready set
      for (size_t i = 0; i < ids.size(); ++i) publish(ids[i]);
      idle.push_back(w);
    }
  }

  void commit(double t) {
    while (!done && head >= 0) {
      Seg& e = segs[head];
      if (del_on && is_prefix(del, e.u)) {  // under a pruned ancestor: skipped
        head = e.next;
        continue;
      }
      del_on = false;
      if (e.st != DONE) break;
      if (e.cut != C) {  // stale: re-run at the exact cutoff, highest priority
        e.st = QUEUED;
        e.pred = C;
        e.rerun_exact = true;
        ready.push_back(head);
        out.reruns++;
        break;
      }
      const RunResult& r = e.res;
      if (pb.budget >= 0 && V + r.visits > pb.budget) {
        // the reference aborts inside this segment: re-run with the exact cap
        RunResult rr = run_segment(pb, e.u, e.end.empty() ? nullptr : &e.end, C, pb.budget - V);
        if (rr.best.has && (!gbest.has || better(rr.best.obj, rr.best.G, gbest.obj, gbest.G)))
          gbest = rr.best;
        V = pb.budget;
        aborted = true;
        done = true;
        now = t + rr.visits;
        break;
      }
      V += r.visits;
      t += prm.commit_cost;
      if (r.best.has && (!gbest.has || better(r.best.obj, r.best.G, gbest.obj, gbest.G)))
        gbest = r.best;
      if (r.m > C) {
        C = r.m;
        if (prm.stale_abort) abort_stale(t);
      }
      const int nxt = e.next;
      if (!e.end.empty() && r.a_star >= 0) {
        del.assign(e.end.begin(), e.end.begin() + r.a_star);
        del_on = true;
      }
      head = nxt;
      if (pb.budget >= 0 && V == pb.budget) {
        // abort iff any further node remains
        int j = head;
        while (j >= 0 && del_on && is_prefix(del, segs[j].u)) j = segs[j].next;
        aborted = j >= 0 || !r.finished;  // a capped run left nodes behind
        done = true;
        break;
      }
    }
    if (head < 0) done = true;
  }

  void abort_stale(double t) {
    for (int s = head; s >= 0; s = segs[s].next) {
      Seg& e = segs[s];
      if (e.st == RUNNING && e.cut < C) {
        out.aborts++;
        out.run_visits += (long long)std::max(0.0, t - e.t0);
        e.gen++;
        e.st = QUEUED;
        e.pred = C;
        idle.push_back(e.warp);
        ready.push_back(s);
      } else if (e.st == DONE && e.cut < C) {  // finished at a stale cutoff: re-run now
        out.reruns++;
        e.st = QUEUED;
        e.pred = C;
        ready.push_back(s);
      }
    }
  }

  Outcome run() {
    // root: its only child [0]; the root node check (grouping.cpp:151-169) is
    // not a visit and happens with the floor cutoff
    GState s0;
    s0.gp.assign(pb.n + 1, 0);
    s0.gm.assign(pb.n + 1, 0);
    s0.gc.assign(pb.n + 1, 0);
    if (node_passes(pb, s0, 0, C)) {
      Seg e;
      e.u = Path{0};
      e.pred = C;
      segs.push_back(e);
      head = 0;
      ready.push_back(0);
    }
    for (int w = 0; w < prm.warps; ++w) idle.push_back(w);
    dispatch(0);
    commit(0);
    request_splits(0);
    tick_pending = true;
    ev.push({std::max(1.0, prm.req_latency), 2, 0, 0});
    while (!done && !ev.empty()) {
      const Event x = ev.top();
      ev.pop();
      Seg& e = segs[x.seg];
      if (x.kind != 2 && x.kind != 5 && x.gen != e.gen) continue;  // superseded
      now = x.t;
      if (x.kind == 5) {  // list merge: pending pieces become dispatchable
        merge_pending = false;
        for (int id : pending) ready.push_back(id);
        pending.clear();
      } else if (x.kind == 2) {  // scheduler tick: re-issue split requests while warps idle
        tick_pending = false;
        if (getenv("ASYNC_EMU_TRACE") && ++ticks % 200 == 0)
          fprintf(stderr, "t=%.0f V=%lld C=%g segs=%zu ready=%zu idle=%zu runs=%lld splits=%lld\n",
                  x.t, V, C, segs.size(), ready.size(), idle.size(), out.runs, out.splits);
      } else if (x.kind == 4) {  // time slice over: preempt (split, all pieces ready)
        if (e.st != RUNNING) continue;
        if (e.split_req) continue;
        split(x.seg, x.t, false);
        if (segs[x.seg].st == RUNNING) continue;  // finished inside the slice
      } else if (x.kind == 3) {  // lazy run evaluation
        if (e.st == RUNNING) extend(x.seg, std::min<long long>(e.cap, 2 * e.horizon));
        continue;
      } else if (x.kind == 0) {
        if (e.st != RUNNING) continue;
        e.st = DONE;
        idle.push_back(e.warp);
      } else {
        if (e.st != RUNNING || !e.split_req) continue;
        split(x.seg, x.t);
      }
      commit(x.t);
      if (done) break;
      dispatch(x.t);
      request_splits(x.t);
      if (!idle.empty() && !tick_pending) {
        tick_pending = true;
        ev.push({x.t + std::max(1.0, prm.req_latency), 2, 0, 0});
      }
    }
    out.best = gbest;
    out.visited = V;
    out.aborted = aborted;
    out.time = now;
    return out;
  }
};

}  // namespace

extern "C" {

int async_emu_search(int n, const double* p, const double* m, int K, double min_mem,
                     long long budget, double floor_obj, int warps, double pop_cost,
                     double split_cost, double req_latency, double commit_cost, int order,
                     int stale_abort, long long min_split, long long slice, long long merge, int* out_rgs, double* out_obj,
                     int* out_has, long long* out_visited, int* out_aborted, double* out_time,
                     long long* out_stats /* runs, run_visits, splits, reruns, aborts */) {
  Problem pb;
  pb.n = n;
  pb.p.assign(p, p + n);
  pb.m.assign(m, m + n);
  pb.K = K;
  pb.min_mem = min_mem;
  pb.budget = budget;
  pb.floor_obj = floor_obj;
  Params prm{warps, pop_cost, split_cost, req_latency, commit_cost, order, stale_abort,
             min_split, slice, merge};
  Sim sim(pb, prm);
  Outcome o = sim.run();
  *out_has = o.best.has ? 1 : 0;
  if (o.best.has) {
    for (int i = 0; i < n; ++i) out_rgs[i] = o.best.rgs[i];
    *out_obj = o.best.obj;
  }
  *out_visited = o.visited;
  *out_aborted = o.aborted ? 1 : 0;
  *out_time = o.time;
  out_stats[0] = o.runs;
  out_stats[1] = o.run_visits;
  out_stats[2] = o.splits;
  out_stats[3] = o.reruns;
  out_stats[4] = o.aborts;
  return 0;
}
}
