/* libspx_sched: native path planner for the SkipPipe scheduler (host C++, no CUDA).
 *
 * The reference specifies its scheduler only in prose (Algorithm 2 at
 * :611-683) -- there is no reference code to bind.  paper_2502_19913_b200/scheduler.py restates
 * it in Python (astar_path, detect_conflicts, the two CBS phases); these entry points are the
 * native form of its two inner loops, called through ctypes by scheduler.py when the library is
 * built (SPX_SCHED_NATIVE=0 forces the Python path).  Results are identical to the Python code.
 *
 * Conventions: return SPX_SCHED_OK (0) on success, SPX_SCHED_INFEASIBLE (1) when no path
 * satisfies the constraints (scheduler.InfeasibleError), negative on bad arguments; no
 * allocation is visible to the caller; no global state. */
#ifndef SPX_SCHED_H
#define SPX_SCHED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPX_SCHED_OK 0
#define SPX_SCHED_INFEASIBLE 1
#define SPX_SCHED_ERR_ARG -1

/* One scheduling problem (scheduler._Timing): n logical nodes, s stages, path length l
 * (PAPER.md:119), node -> stage, per-node forward / backward compute ms, comm ms [n][n]
 * (topology.comm_matrix at the message size; topology.py:139-147). */
typedef struct {
  int32_t n, s, l, max_swaps;
  const int32_t* node_stage;
  const double* fwd;
  const double* bwd;
  const double* comm;
} spx_sched_problem;

int spx_sched_abi_version(void);

/* scheduler.astar_path for the agent starting at `origin`: minimum-e2e route under CC1 / CC2 /
 * exact-l and the agent's interval constraints (cnode[i] unavailable during [ct0[i], ct1[i]];
 * (-inf, +inf) bans the node); require_swap = SchedulerConfig.swap_agents membership.
 * Outputs: out_nodes[len] (origin first), out_fwd[(len+1)*3] (arrival, start, end per forward
 * visit, then the return visit), out_bwd[len*3] (backward visits in execution order),
 * out_swaps, out_e2e.  Buffers must hold s nodes / (s+1)*3 and s*3 doubles. */
int spx_sched_astar(const spx_sched_problem* p, int32_t origin, int32_t require_swap, int32_t ncons,
                    const int32_t* cnode, const double* ct0, const double* ct1, int32_t* out_nodes, double* out_fwd,
                    double* out_bwd, int32_t* out_len, int32_t* out_swaps, double* out_e2e);

/* Forward-interval collisions of a CBS node (scheduler.detect_conflicts): agents
 * sorted by id, cnt[k] visits each as (vnode, vstart, vend).  Writes up to max_out collisions
 * (agent_i < agent_j, node) and (lo, hi, s_i, e_i, s_j, e_j); returns how many exist. */
int64_t spx_sched_collisions(int32_t n_agents, const int32_t* agent_ids, const int32_t* cnt, const int32_t* vnode,
                             const double* vstart, const double* vend, int32_t n_nodes, int64_t max_out,
                             int32_t* out_ij_node, double* out_times);

#ifdef __cplusplus
}
#endif

#endif
