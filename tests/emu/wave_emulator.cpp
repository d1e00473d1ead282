// wave_emulator.cpp — CPU emulation of the B200 grouping scheduler (design
// validation harness; NOT product code, never linked into the library).
//
// It runs the exact algorithm the CUDA kernel runs — ordered segment list,
// speculative waves at the front cutoff, speculative splitting of unfinished
// segments into [prefix record] + [remainder pieces], the ordered commit walk,
// prefix re-runs with an end marker and ancestor-prune deletion, and the
// budget cut through per-segment improvement logs — but with a serial segment
// runner. tests/test_scheduler_emulator.py checks it against the oracle
// (oracle/hetplan_oracle.c) on thousands of random instances with tiny caps so
// that every scheduler path is exercised. See DESIGN.md "Grouping search".
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

static bool better(double ao, int ag, double bo, int bg) {
  if (ao != bo) return ao > bo;
  return ag < bg;
}

struct Event {
  long long visit;  // 1-based visit index within the run
  double obj;
  int G;
};

struct RunResult {
  long long visits = 0;
  bool finished = false;  // subtree exhausted / end marker reached
  Path stop;              // next node to enter when !finished
  Best best;
  std::vector<Event> events;
  double m = -1;          // max feasible-leaf objective seen (-1 none)
  int a_star = -1;        // prefix re-runs: depth of the pruned ancestor of the end marker
};

// Group state of a prefix path.
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

// The node check of P/src/grouping.cpp:151-169, exact serial order.
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

// Preorder position compare of paths: -1 if a<b, 0 eq, 1 if a>b (ancestor < descendant).
int path_cmp(const Path& a, const Path& b) {
  const size_t k = a.size() < b.size() ? a.size() : b.size();
  for (size_t i = 0; i < k; ++i) {
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  }
  if (a.size() == b.size()) return 0;
  return a.size() < b.size() ? -1 : 1;
}

bool is_prefix(const Path& a, const Path& b) {  // a is a prefix of b (ancestor or equal)
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

// Segment runner: DFS of subtree(u) in preorder starting at node `start`
// (entered first), stopping after `cap` visits, or before entering a node >=
// `end` (if non-empty). Exact reference semantics per node.
RunResult run_segment(const Problem& pb, const Path& u, const Path& start, const Path* end,
                      double cutoff, long long cap) {
  RunResult r;
  GState s;
  s.gp.assign(pb.n + 1, 0);
  s.gm.assign(pb.n + 1, 0);
  s.gc.assign(pb.n + 1, 0);
  Path cur;  // path of the last entered/being-processed node
  // Set up ancestors of start.
  for (size_t i = 0; i + 1 < start.size(); ++i) {
    apply(pb, s, (int)i, start[i]);
    cur.push_back(start[i]);
  }
  // `next` = node to enter next (as a path). We iterate: enter next; process.
  Path next = start;
  bool have_next = true;
  double c = cutoff;
  auto advance_from = [&](Path x) -> bool {
    // x processed with its subtree done (or pruned). Find next sibling upward,
    // staying inside subtree(u). State `s` reflects x applied; undo as we go up.
    while (true) {
      if (x.size() == u.size()) return false;  // subtree(u) exhausted
      const int d = (int)x.size() - 1;
      const int g = x[d];
      undo(pb, s, d, g);
      cur.pop_back();
      const int Gp = s.G;  // groups of parent
      if (g + 1 <= Gp) {
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
      r.finished = false;
      r.stop = next;
      return r;
    }
    // enter next
    r.visits++;
    const int d = (int)next.size() - 1;
    apply(pb, s, d, next[d]);
    cur.push_back(next[d]);
    Path x = next;
    if ((int)x.size() == pb.n) {  // leaf
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
          r.events.push_back({r.visits, obj, s.G});
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

enum Kind { FULL, PREFIX };

struct Entry {
  Kind kind = FULL;
  Path u;        // root (entered by this entry)
  Path end;      // PREFIX: end marker
  bool ran = false;
  double cutoff_used = 0;
  RunResult res;
};

struct Outcome {
  Best best;
  long long visited = 0;
  bool aborted = false;
  int waves = 0;
  long long runs = 0, run_visits = 0;
  int max_list = 0;
};

// Remainder pieces of subtree(u) after stop point q (q inside subtree(u)):
// subtree(q), then right siblings of q's ancestors up to u's depth.
void remainder_pieces(const Path& u, const Path& q, std::vector<Entry>& out) {
  Entry e;
  e.u = q;
  out.push_back(e);
  for (int d = (int)q.size() - 1; d >= (int)u.size(); --d) {
    const int Gp = groups_of(q, d);
    for (int c = q[d] + 1; c <= Gp; ++c) {
      Entry s;
      s.u.assign(q.begin(), q.begin() + d);
      s.u.push_back((uint8_t)c);
      out.push_back(s);
    }
  }
}

Outcome schedule(const Problem& pb, int nw, long long cap, int max_list) {
  Outcome out;
  // Root (not a visit): check, then its only child [0].
  GState s0;
  s0.gp.assign(pb.n + 1, 0);
  s0.gm.assign(pb.n + 1, 0);
  s0.gc.assign(pb.n + 1, 0);
  double C = pb.floor_obj;
  std::vector<Entry> list;
  if (node_passes(pb, s0, 0, C)) {
    Entry e;
    e.u = Path{0};
    list.push_back(e);
  }
  long long V = 0;
  Best gbest;
  const long long B = pb.budget;
  while (!list.empty()) {
    out.waves++;
    out.max_list = (int)list.size() > out.max_list ? (int)list.size() : out.max_list;
    // Run phase: first nw entries that need a run at cutoff C.
    int launched = 0;
    for (size_t i = 0; i < list.size() && launched < nw; ++i) {
      Entry& e = list[i];
      if (e.ran && e.cutoff_used == C) continue;
      e.ran = true;
      e.cutoff_used = C;
      if (e.kind == FULL) {
        e.res = run_segment(pb, e.u, e.u, nullptr, C, cap);
      } else {
        e.res = run_segment(pb, e.u, e.u, &e.end, C, (long long)1 << 62);
      }
      launched++;
      out.runs++;
      out.run_visits += e.res.visits;
    }
    // Split phase: unfinished FULL runs -> PREFIX record + remainder pieces.
    {
      std::vector<Entry> nl;
      nl.reserve(list.size() * 2);
      int budget_left = max_list - (int)list.size();
      bool first = true;
      for (auto& e : list) {
        const bool front = first;  // the front entry always splits (progress guarantee)
        first = false;
        if (e.kind == FULL && e.ran && !e.res.finished) {
          std::vector<Entry> pieces;
          remainder_pieces(e.u, e.res.stop, pieces);
          if (front || (int)pieces.size() <= budget_left) {
            budget_left -= (int)pieces.size();
            Entry rec = e;
            rec.kind = PREFIX;
            rec.end = e.res.stop;
            rec.res.finished = true;
            nl.push_back(rec);
            for (auto& pc : pieces) nl.push_back(pc);
            continue;
          }
          // no room: discard the partial run (re-run next wave)
          e.ran = false;
        }
        nl.push_back(e);
      }
      list.swap(nl);
    }
    // Commit walk.
    size_t i = 0;
    bool done = false;
    while (i < list.size()) {
      Entry& e = list[i];
      if (!e.ran || e.cutoff_used != C || !e.res.finished) break;
      const RunResult& r = e.res;
      if (B >= 0 && V + r.visits > B) {
        // Budget runs out inside this entry at local visit v*.
        const long long vstar = B - V;
        const Event* last = nullptr;
        for (const auto& ev : r.events)
          if (ev.visit <= vstar) last = &ev;
        if (last) {
          Best lb;
          lb.has = true;
          lb.obj = last->obj;
          lb.G = last->G;
          if (last == &r.events.back()) {
            lb.rgs = r.best.rgs;
          } else {
            RunResult rr = run_segment(pb, e.u, e.u, e.kind == PREFIX ? &e.end : nullptr,
                                       C, vstar);
            lb.rgs = rr.best.rgs;
          }
          if (!gbest.has || better(lb.obj, lb.G, gbest.obj, gbest.G)) gbest = lb;
        }
        V = B;
        out.aborted = true;
        done = true;
        break;
      }
      V += r.visits;
      if (r.best.has && (!gbest.has || better(r.best.obj, r.best.G, gbest.obj, gbest.G)))
        gbest = r.best;
      if (r.m > C) C = r.m;
      size_t j = i + 1;
      if (e.kind == PREFIX && r.a_star >= 0) {
        Path anc(e.end.begin(), e.end.begin() + r.a_star);
        while (j < list.size() && is_prefix(anc, list[j].u)) ++j;
      }
      // V == B: abort iff any further node will be attempted.
      if (B >= 0 && V == B && j < list.size()) {
        out.aborted = true;
        done = true;
        break;
      }
      i = j;
    }
    if (done) break;
    list.erase(list.begin(), list.begin() + i);
  }
  out.best = gbest;
  out.visited = V;
  return out;
}

}  // namespace

extern "C" {

// Returns the emulated search. Inputs mirror hpo_solve_grouping minus seeds
// (the caller passes the seed objective as floor_obj). rgs out is the best
// partition (n ints), or untouched if none found.
int emu_search(int n, const double* p, const double* m, int K, double min_mem,
               long long budget, double floor_obj, int nw, long long cap, int max_list,
               int* out_rgs, double* out_obj, int* out_has, long long* out_visited,
               int* out_aborted, int* out_waves, long long* out_runs,
               long long* out_run_visits, int* out_max_list) {
  Problem pb;
  pb.n = n;
  pb.p.assign(p, p + n);
  pb.m.assign(m, m + n);
  pb.K = K;
  pb.min_mem = min_mem;
  pb.budget = budget;
  pb.floor_obj = floor_obj;
  Outcome o = schedule(pb, nw, cap, max_list);
  *out_has = o.best.has ? 1 : 0;
  if (o.best.has) {
    for (int i = 0; i < n; ++i) out_rgs[i] = o.best.rgs[i];
    *out_obj = o.best.obj;
  }
  *out_visited = o.visited;
  *out_aborted = o.aborted ? 1 : 0;
  *out_waves = o.waves;
  *out_runs = o.runs;
  *out_run_visits = o.run_visits;
  *out_max_list = o.max_list;
  return 0;
}
}
