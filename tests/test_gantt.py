"""SVG Gantt / trace CSV artifacts on simulated timelines."""

import xml.etree.ElementTree as ET

import pytest

from paper_2502_19913_b200.configs import get_config
from paper_2502_19913_b200.errors import ValidationError
from paper_2502_19913_b200.gantt import emit_gantt, intervals, trace_csv
from paper_2502_19913_b200.simulator import SimReport, simulate

NS = "{http://www.w3.org/2000/svg}"


def _sim(name="C1"):
    rc = get_config(name)
    return rc, simulate(rc.schedule(), rc.topology(), rc.sim_config(record_trace=True))


def test_gantt_one_rect_per_compute_interval():
    rc, rep = _sim()
    svg = emit_gantt(rep, rc.topology().n, "C1")
    root = ET.fromstring(svg)  # well-formed standalone SVG
    titled = [r for r in root.iter(NS + "rect") if r.find(NS + "title") is not None]
    assert len(titled) == len(rep.ops) == len(rep.trace) // 2
    # node bands: one background row per node
    assert sum(1 for t in root.iter(NS + "text") if (t.text or "").startswith("node ")) == rc.topology().n


def test_intervals_match_ops_and_order():
    rc, rep = _sim()
    iv = intervals(rep.trace)
    assert len(iv) == len(rep.ops)
    per_node = {}
    for node, t0, t1, agent, wave, d in sorted(iv, key=lambda r: (r[0], r[1])):
        assert t1 >= t0
        per_node.setdefault(node, []).append((t0, t1))
    for node, spans in per_node.items():  # a node runs one op at a time
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert b0 >= a1 - 1e-9


def test_trace_csv_header_and_rows():
    _, rep = _sim()
    lines = trace_csv(rep.trace).splitlines()
    assert lines[0] == "time_ms,node,event,agent,wave,direction"
    assert len(lines) == 1 + len(rep.trace)


def test_empty_trace_and_missing_trace():
    empty = SimReport(iteration_makespan=0.0, microbatch_e2e=[], total_collision_wait=0.0, node_busy=[0.0] * 3,
                      node_idle=[0.0] * 3, ops=[], trace=[])
    root = ET.fromstring(emit_gantt(empty))
    assert not [r for r in root.iter(NS + "rect") if r.find(NS + "title") is not None]
    assert sum(1 for t in root.iter(NS + "text") if (t.text or "").startswith("node ")) == 3
    empty.trace = None
    with pytest.raises(ValidationError, match="--trace"):
        emit_gantt(empty)
