"""Timeline artifacts: trace CSV rows and the SVG Gantt chart.

``emit_gantt`` renders any report that carries a trace -- the simulator's planned timeline
(``SimReport``, recorded with ``SimConfig(record_trace=True)``) or the executor's measured one
(``ExecReport`` from ``Trainer.make_report``, CUDA-event times, rows from every rank merged) --
as one horizontal band per logical node and one rectangle per compute interval, labelled
(agent, wave, direction), on a time axis in ms.  Colours follow the agent (microbatch stream);
backward is drawn darker than forward, the loss op at the origin hatched-dark.
"""

from __future__ import annotations

import csv
import io
from xml.sax.saxutils import escape

from .errors import ValidationError

_PALETTE = ["#4e79a7", "#f28e2b", "#e15759", "#76b7b2", "#59a14f", "#edc948", "#b07aa1", "#ff9da7",
            "#9c755f", "#bab0ac"]


def trace_csv(trace) -> str:
    """Trace rows (time_ms, node, event, agent, wave, direction) as CSV text."""
    if trace is None:
        raise ValidationError("report was recorded without a trace; rerun with record_trace=True (--trace)")
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["time_ms", "node", "event", "agent", "wave", "direction"])
    for row in trace:
        w.writerow([repr(float(row[0])), *row[1:]])
    return buf.getvalue()


def intervals(trace) -> list[tuple[int, float, float, int, int, str]]:
    """Pair start/end rows into compute intervals (node, t0, t1, agent, wave, direction)."""
    open_: dict[tuple, float] = {}
    out = []
    for t, node, event, agent, wave, direction in sorted(trace, key=lambda r: (r[0], r[2] != "end")):
        key = (node, agent, wave, direction)
        if event == "start":
            open_[key] = float(t)
        elif event == "end":
            if key not in open_:
                raise ValidationError(f"trace: end without start for node {node}, agent {agent}, wave {wave}, "
                                      f"{direction}")
            out.append((int(node), open_.pop(key), float(t), int(agent), int(wave), str(direction)))
    if open_:
        raise ValidationError(f"trace: {len(open_)} intervals never end")
    return out


def emit_gantt(report, n_nodes: int | None = None, title: str = "", width: int = 1400) -> str:
    """Standalone SVG Gantt chart of ``report.trace``."""
    trace = getattr(report, "trace", None)
    if trace is None:
        raise ValidationError("report was recorded without a trace; rerun with record_trace=True (--trace)")
    iv = intervals(trace)
    nodes = n_nodes if n_nodes is not None else (max((r[0] for r in iv), default=-1) + 1)
    nodes = max(nodes, len(getattr(report, "node_busy", []) or []))
    t_end = max([r[2] for r in iv] + [float(getattr(report, "iteration_makespan", 0.0) or 0.0), 1e-9])
    left, top, row_h, gap = 70, 40 if title else 20, 28, 6
    plot_w = width - left - 20
    height = top + nodes * (row_h + gap) + 40
    sx = plot_w / t_end

    def x(t: float) -> float:
        return left + t * sx

    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width}" height="{height}" '
           f'viewBox="0 0 {width} {height}" font-family="sans-serif" font-size="10">',
           '<defs><pattern id="loss" width="4" height="4" patternUnits="userSpaceOnUse">'
           '<path d="M0,4 L4,0" stroke="#000" stroke-width="1"/></pattern></defs>']
    if title:
        out.append(f'<text x="{left}" y="16" font-size="13">{escape(title)}</text>')
    for v in range(nodes):
        y = top + v * (row_h + gap)
        out.append(f'<rect x="{left}" y="{y}" width="{plot_w}" height="{row_h}" fill="#f4f4f4"/>')
        out.append(f'<text x="{left - 8}" y="{y + row_h * 0.65}" text-anchor="end">node {v}</text>')
    # time axis
    y_ax = top + nodes * (row_h + gap) + 4
    out.append(f'<line x1="{left}" y1="{y_ax}" x2="{left + plot_w}" y2="{y_ax}" stroke="#333"/>')
    step = _nice_step(t_end / 10)
    t = 0.0
    while t <= t_end + 1e-9:
        out.append(f'<line x1="{x(t):.2f}" y1="{y_ax}" x2="{x(t):.2f}" y2="{y_ax + 4}" stroke="#333"/>')
        out.append(f'<text x="{x(t):.2f}" y="{y_ax + 15}" text-anchor="middle">{t:g}</text>')
        t += step
    out.append(f'<text x="{left + plot_w}" y="{y_ax + 28}" text-anchor="end">time (ms)</text>')
    for node, t0, t1, agent, wave, direction in sorted(iv, key=lambda r: (r[0], r[1])):
        y = top + node * (row_h + gap)
        col = _PALETTE[agent % len(_PALETTE)]
        op = {"fwd": 0.55, "bwd": 1.0, "loss": 1.0}.get(direction, 0.8)
        w = max((t1 - t0) * sx, 0.5)
        label = f"a{agent} w{wave} {direction}"
        out.append(f'<rect x="{x(t0):.2f}" y="{y + 2}" width="{w:.2f}" height="{row_h - 4}" fill="{col}" '
                   f'fill-opacity="{op}" stroke="#222" stroke-width="0.3"><title>{escape(label)} '
                   f'[{t0:.3f}, {t1:.3f}] ms</title></rect>')
        if direction == "loss":
            out.append(f'<rect x="{x(t0):.2f}" y="{y + 2}" width="{w:.2f}" height="{row_h - 4}" fill="url(#loss)" '
                       f'fill-opacity="0.5"/>')
        if w > 38:
            out.append(f'<text x="{x(t0) + 2:.2f}" y="{y + row_h * 0.65}" font-size="8">{escape(label)}</text>')
    out.append("</svg>")
    return "\n".join(out)


def _nice_step(raw: float) -> float:
    if raw <= 0:
        return 1.0
    import math

    e = 10 ** math.floor(math.log10(raw))
    for m in (1, 2, 5, 10):
        if raw <= m * e:
            return m * e
    return 10 * e
