"""Native path planner (libspx_sched.so, include/spx_sched.h) against the
Python restatement in scheduler.py: identical A* plans (routes, visit times, swaps, e2e) on 300
random instances with random interval constraints and bans, identical conflict lists, and
identical end-to-end schedules for the BASELINE configs."""

import math
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2502_19913_b200 import scheduler as S
from paper_2502_19913_b200.configs import get_config
from paper_2502_19913_b200.allocation import StageAssignment
from paper_2502_19913_b200.errors import InfeasibleError
from paper_2502_19913_b200.topology import Topology

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    so = os.path.join(ROOT, "paper_2502_19913_b200", "libspx_sched.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", ROOT, "sched"], check=True)
    assert S.native_lib() is not None


def _random_instance(rng, n_max=8, s_max=4):
    s = int(rng.integers(2, s_max + 1))
    sizes = [1] + [int(x) for x in rng.integers(1, 3, size=s - 1)]
    while sum(sizes) > n_max:
        sizes[int(np.argmax(sizes))] -= 1
    n = sum(sizes)
    T = Topology(n=n, latency_ms=rng.uniform(1, 20, size=(n, n)), bandwidth_bytes_per_ms=rng.uniform(1e5, 1e6, size=(n, n)),
                 compute_fwd_ms=rng.uniform(5, 50, size=n), bwd_ratio=float(rng.uniform(1, 3)))
    l = int(rng.integers(2, s + 1))
    return T, StageAssignment.contiguous(sizes), 100 * (s - l) / s, l


def _both(fn, monkeypatch):
    monkeypatch.setenv("SPX_SCHED_NATIVE", "1")
    try:
        a = ("ok", fn())
    except InfeasibleError as e:
        a = ("infeasible", str(e))
    monkeypatch.setenv("SPX_SCHED_NATIVE", "0")
    try:
        b = ("ok", fn())
    except InfeasibleError as e:
        b = ("infeasible", str(e))
    monkeypatch.setenv("SPX_SCHED_NATIVE", "1")
    return a, b


def test_header_symbols_exported():
    txt = open(os.path.join(ROOT, "include", "spx_sched.h")).read()
    syms = re.findall(r"^\s*(?:int|int64_t)\s+(spx_sched_\w+)\s*\(", txt, flags=re.M)
    lib = S.native_lib()
    assert len(syms) == 3 and all(hasattr(lib, x) for x in syms)
    assert lib.spx_sched_abi_version() == 1


def test_astar_native_equals_python(monkeypatch):
    rng = np.random.default_rng(99)
    checked = 0
    for it in range(300):
        T, A, k, l = _random_instance(rng)
        swap = () if it % 3 else (0,)
        cfg = S.SchedulerConfig(k=k, msg_bytes=1e6, swap_agents=swap)
        cons = []
        for _ in range(int(rng.integers(0, 4))):
            v = int(rng.integers(0, T.n))
            if rng.random() < 0.3:
                cons.append(S.IntervalConstraint(0, v, -math.inf, math.inf))
            else:
                t0 = float(rng.uniform(0, 200))
                cons.append(S.IntervalConstraint(0, v, t0, t0 + float(rng.uniform(1, 80))))
        a, b = _both(lambda: S.astar_path(S.Agent(0, 0), T, A, tuple(cons), cfg), monkeypatch)
        assert a == b, (it, a, b)
        checked += a[0] == "ok"
    assert checked > 150


def test_conflicts_native_equal_python(monkeypatch):
    for name in ("C1", "C2", "C3"):
        rc = get_config(name)
        sch = rc.schedule()
        node = S.SearchNode(frozenset(), dict(sch.paths), sch.cost_ms)
        a, b = _both(lambda: S.detect_conflicts(node, rc.topology(), rc.assignment, 1, k=rc.k), monkeypatch)
        assert a == b


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5", "C2-rb"])
def test_schedules_identical(name, monkeypatch):
    def run():
        rc = get_config(name)
        return rc.schedule().to_dict()

    a, b = _both(run, monkeypatch)
    assert a == b
