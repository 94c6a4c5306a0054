// Native path planner for the SkipPipe scheduler: the time-dimensioned A*
// of one agent under CC1 / CC2 / exact-l and its interval constraints (SPEC.md:237-246,
// PAPER.md:245-267), and the conflict scan of a CBS node's paths.  Host-only
// C++ (no CUDA), behind the C-ABI in include/spx_sched.h; scheduler.py's CBS calls it for every
// (re)plan and conflict check.  Results are identical to the Python restatement: same float64
// operation order (built with -ffp-contract=off), same heap tie-breaking as Python's tuple order
// (cost, node, time, node sequence, completion flag).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <vector>

#include "../../include/spx_sched.h"

namespace {

struct Visit {
  int node, stage;
  double arr, start, end;
};

struct Entry {
  double cost;
  int u;
  double t;
  std::vector<int> nodes;
  int flagged;
  // payload
  std::vector<int> seq;
  int swaps;
  std::vector<Visit> visits;  // forward visits (flagged: + return visit)
  std::vector<Visit> bwd;     // flagged only
};

// Python tuple order (cost, agent, u, t, nodes, flagged, ...): a > b for a min-heap
struct Greater {
  bool operator()(const Entry* a, const Entry* b) const {
    if (a->cost != b->cost) return a->cost > b->cost;
    if (a->u != b->u) return a->u > b->u;
    if (a->t != b->t) return a->t > b->t;
    if (a->nodes != b->nodes) return a->nodes > b->nodes;  // lexicographic, prefix smaller
    return a->flagged > b->flagged;
  }
};

struct Windows {
  std::vector<std::vector<std::pair<double, double>>> w;  // per node, sorted
  double start_at(int node, double t, double dur) const {
    const auto& ws = w[node];
    if (ws.empty()) return t;
    bool moved = true;
    while (moved) {
      moved = false;
      for (const auto& p : ws) {
        if (t < p.second && p.first < t + dur) {
          t = p.second;
          moved = true;
        }
      }
    }
    return t;
  }
};

// CC2: returns the swap count after appending x, or -1 if forbidden
int cc2_extend(const std::vector<int>& seq, int swaps, int x, int max_swaps) {
  int mx = seq[0];
  for (int v : seq) {
    if (v == x) return -1;
    mx = std::max(mx, v);
  }
  if (x > mx) return swaps;
  if (swaps >= max_swaps || seq.size() < 2) return -1;
  if (seq[seq.size() - 2] < x && x < seq.back()) return swaps + 1;
  return -1;
}

}  // namespace

extern "C" int spx_sched_abi_version(void) { return 1; }

extern "C" int spx_sched_astar(const spx_sched_problem* p, int32_t origin, int32_t require_swap, int32_t ncons,
                               const int32_t* cnode, const double* ct0, const double* ct1, int32_t* out_nodes,
                               double* out_fwd, double* out_bwd, int32_t* out_len, int32_t* out_swaps,
                               double* out_e2e) {
  if (!p || !p->node_stage || !p->fwd || !p->bwd || !p->comm || !out_nodes || !out_fwd || !out_bwd || !out_len ||
      !out_swaps || !out_e2e)
    return SPX_SCHED_ERR_ARG;
  const int n = p->n, s = p->s, l = p->l;
  if (n <= 0 || s <= 0 || l <= 0 || l > s || origin < 0 || origin >= n || ncons < 0) return SPX_SCHED_ERR_ARG;
  if (p->node_stage[origin] != 0) return SPX_SCHED_ERR_ARG;
  std::vector<char> banned(n, 0);
  Windows win;
  win.w.resize(n);
  for (int i = 0; i < ncons; ++i) {
    const int v = cnode[i];
    if (v < 0 || v >= n) return SPX_SCHED_ERR_ARG;
    if (std::isinf(ct0[i]) && ct0[i] < 0 && std::isinf(ct1[i]) && ct1[i] > 0) banned[v] = 1;
    else win.w[v].emplace_back(ct0[i], ct1[i]);
  }
  for (auto& ws : win.w) std::sort(ws.begin(), ws.end());
  if (banned[origin]) return SPX_SCHED_INFEASIBLE;
  std::vector<std::vector<int>> stage_nodes(s);
  for (int v = 0; v < n; ++v) stage_nodes[p->node_stage[v]].push_back(v);
  const double* comm = p->comm;
  auto C = [&](int a, int b) { return comm[(size_t)a * n + b]; };

  std::vector<Entry*> pool;
  std::priority_queue<Entry*, std::vector<Entry*>, Greater> heap;
  auto push = [&](Entry* e) {
    pool.push_back(e);
    heap.push(e);
  };
  {
    const double st0 = win.start_at(origin, 0.0, p->fwd[origin]);
    Entry* e = new Entry{st0 + p->fwd[origin], origin, st0 + p->fwd[origin], {origin}, 0, {0}, 0,
                         {{origin, 0, 0.0, st0, st0 + p->fwd[origin]}}, {}};
    push(e);
  }
  int rc = SPX_SCHED_INFEASIBLE;
  while (!heap.empty()) {
    Entry* e = heap.top();
    heap.pop();
    if (e->flagged) {
      const int k = (int)e->nodes.size();
      for (int i = 0; i < k; ++i) out_nodes[i] = e->nodes[i];
      for (int i = 0; i <= k; ++i) {
        out_fwd[3 * i] = e->visits[i].arr;
        out_fwd[3 * i + 1] = e->visits[i].start;
        out_fwd[3 * i + 2] = e->visits[i].end;
      }
      for (int i = 0; i < k; ++i) {
        out_bwd[3 * i] = e->bwd[i].arr;
        out_bwd[3 * i + 1] = e->bwd[i].start;
        out_bwd[3 * i + 2] = e->bwd[i].end;
      }
      *out_len = k;
      *out_swaps = e->swaps;
      *out_e2e = e->cost;
      rc = SPX_SCHED_OK;
      break;
    }
    const int u = e->u;
    const double t = e->t;
    if ((int)e->seq.size() == l) {
      if (e->swaps == 0 && require_swap) continue;
      const double t_ret = t + (u != origin ? C(u, origin) : 0.0);
      // backward plan (mirrored route, the agent's own windows delay it too)
      std::vector<Visit> bw;
      double tb = t_ret;
      int prev = origin;
      for (int i = (int)e->nodes.size() - 1; i >= 1; --i) {
        const int v = e->nodes[i];
        const double arr = tb + C(prev, v);
        const double st = win.start_at(v, arr, p->bwd[v]);
        tb = st + p->bwd[v];
        bw.push_back({v, p->node_stage[v], arr, st, tb});
        prev = v;
      }
      const double arr = tb + (prev != origin ? C(prev, origin) : 0.0);
      const double st = win.start_at(origin, arr, p->bwd[origin]);
      tb = st + p->bwd[origin];
      bw.push_back({origin, 0, arr, st, tb});
      Entry* f = new Entry{tb, origin, t_ret, e->nodes, 1, e->seq, e->swaps, e->visits, std::move(bw)};
      f->visits.push_back({origin, 0, t_ret, t_ret, t_ret});
      push(f);
      continue;
    }
    for (int x = 1; x < s; ++x) {
      const int ns = cc2_extend(e->seq, e->swaps, x, p->max_swaps);
      if (ns < 0) continue;
      for (int v : stage_nodes[x]) {
        if (banned[v]) continue;
        const double arr = t + C(u, v);
        const double st = win.start_at(v, arr, p->fwd[v]);
        const double end = st + p->fwd[v];
        Entry* c = new Entry{end, v, end, e->nodes, 0, e->seq, ns, e->visits, {}};
        c->nodes.push_back(v);
        c->seq.push_back(x);
        c->visits.push_back({v, x, arr, st, end});
        push(c);
      }
    }
  }
  for (Entry* e : pool) delete e;
  return rc;
}

// Forward-interval collisions among a CBS node's paths: every pair of different
// agents whose planned compute intervals on one node overlap.  paths are given as flat arrays:
// agent ids (sorted ascending), per agent k its visit count cnt[k] and (node, start, end) triples.
// Writes up to max_out collisions as (agent_i, agent_j, node, lo, hi, s_i, e_i, s_j, e_j) with
// i < j, in the Python enumeration order (node ascending, then the pair order of the per-node
// interval list built agent by agent); returns the number found (may exceed max_out).
extern "C" int64_t spx_sched_collisions(int32_t n_agents, const int32_t* agent_ids, const int32_t* cnt,
                                        const int32_t* vnode, const double* vstart, const double* vend, int32_t n_nodes,
                                        int64_t max_out, int32_t* out_ij_node, double* out_times) {
  if (n_agents < 0 || n_nodes <= 0) return SPX_SCHED_ERR_ARG;
  struct Iv {
    int a;
    double s, e;
  };
  std::vector<std::vector<Iv>> by_node(n_nodes);
  int64_t off = 0;
  for (int k = 0; k < n_agents; ++k) {
    for (int i = 0; i < cnt[k]; ++i, ++off) {
      const int v = vnode[off];
      if (v < 0 || v >= n_nodes) return SPX_SCHED_ERR_ARG;
      by_node[v].push_back({agent_ids[k], vstart[off], vend[off]});
    }
  }
  int64_t found = 0;
  for (int v = 0; v < n_nodes; ++v) {
    const auto& iv = by_node[v];
    for (size_t x = 0; x < iv.size(); ++x)
      for (size_t y = x + 1; y < iv.size(); ++y) {
        const Iv &A = iv[x], &B = iv[y];
        if (A.a == B.a) continue;
        const double lo = std::max(A.s, B.s), hi = std::min(A.e, B.e);
        if (lo < hi) {
          if (found < max_out) {
            const bool ab = A.a < B.a;
            const Iv& I = ab ? A : B;
            const Iv& J = ab ? B : A;
            out_ij_node[3 * found] = I.a;
            out_ij_node[3 * found + 1] = J.a;
            out_ij_node[3 * found + 2] = v;
            double* o = out_times + 6 * found;
            o[0] = lo;
            o[1] = hi;
            o[2] = I.s;
            o[3] = I.e;
            o[4] = J.s;
            o[5] = J.e;
          }
          ++found;
        }
      }
  }
  return found;
}
