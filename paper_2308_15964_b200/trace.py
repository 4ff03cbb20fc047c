"""Dot and SVG export (reference src/trace.py:87-310).

Dot uses the reference dialect exactly (``digraph taskgraph {``, one
``t<tid> [label=...]`` node per task, ``t<src> -> t<dst>`` edges sorted by
pair; reference tests/conftest.py:206-226 parses it).  Edges come from the
native dependency core's slot lists.  The SVG timeline has one lane per
(device, stream) with task rectangles from CUDA-event timestamps and the
ready-count curve from Push/Pop events.
"""

from __future__ import annotations


def _dot_quote(text: str) -> str:
    return '"' + text.replace("\\", "\\\\").replace('"', '\\"') + '"'


def render_dot(graph, show_deps: bool = False) -> str:
    lines = ["digraph taskgraph {"]
    for tid in graph.all_task_ids():
        lines.append(f"  t{tid} [label={_dot_quote(graph._label(tid))}];")
    by_pair = {}
    for src, dst, hid in graph.edges():
        by_pair.setdefault((src, dst), set()).add(hid)
    for (src, dst) in sorted(by_pair):
        if show_deps:
            label = ",".join(f"h{h}" for h in sorted(by_pair[(src, dst)]))
            lines.append(f"  t{src} -> t{dst} [label={_dot_quote(label)}];")
        else:
            lines.append(f"  t{src} -> t{dst};")
    lines.append("}")
    return "\n".join(lines) + "\n"


def generate_dot(graph, path=None, show_deps: bool = False) -> str:
    text = render_dot(graph, show_deps)
    if path is not None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
    return text


def build_lanes(events):
    """Per-worker task intervals [(start, end, tid)] (trace.py:149-160)."""
    lanes = {}
    open_task = {}
    for kind, t, wid, tid, _ in events:
        if kind == "TaskStart":
            open_task[(wid, tid)] = t
        elif kind == "TaskEnd":
            started = open_task.pop((wid, tid), None)
            if started is not None:
                lanes.setdefault(wid, []).append((started, t, tid))
    for v in lanes.values():
        v.sort()
    return lanes


def build_ready_steps(events):
    """Step function [(t, count)] of queued tasks (trace.py:163-174)."""
    steps = [(0, 0)]
    count = 0
    for kind, t, _, _, _ in events:
        if kind == "Push":
            count += 1
            steps.append((t, count))
        elif kind == "Pop":
            count -= 1
            steps.append((t, count))
    return steps


def _union_ns(intervals):
    """Total length of the union of [start, end] intervals (group members share one
    start/end pair, and launch groups on one stream may overlap their waits)."""
    total, cur_s, cur_e = 0, None, None
    for start, end in sorted(intervals):
        if cur_e is None or start > cur_e:
            if cur_e is not None:
                total += cur_e - cur_s
            cur_s, cur_e = start, end
        else:
            cur_e = max(cur_e, end)
    if cur_e is not None:
        total += cur_e - cur_s
    return total


def idle_report(graph, events=None):
    """Per-lane and per-GPU idle time (reference trace.py:292-300 prints one idle
    scalar per worker; a lane here is one CUDA stream of one GPU, and a GPU is
    busy while any of its streams runs a task).  Times from the tasks' CUDA
    start/end events; span = first to last event of the graph.  Returns
    {"span_ms", "lanes": {label: (busy_ms, idle_ms)}, "gpus": {d: (busy_ms, idle_ms)}}."""
    events = graph.trace.export_events() if events is None else events
    lanes = build_lanes(events)
    t_lo = min([e[1] for e in events], default=0)
    t_hi = max([e[1] for e in events], default=0)
    span = max(t_hi - t_lo, 1)
    nstreams = graph.engine.worker_stride() if graph.engine else 1
    out = {"span_ms": span / 1e6, "lanes": {}, "gpus": {}}
    per_dev = {}
    for wid in sorted(lanes):
        iv = [(a, b) for a, b, _ in lanes[wid]]
        busy = _union_ns(iv)
        out["lanes"][f"gpu{wid // nstreams} s{wid % nstreams}"] = (busy / 1e6, (span - busy) / 1e6)
        per_dev.setdefault(wid // nstreams, []).extend(iv)
    for d, iv in sorted(per_dev.items()):
        busy = _union_ns(iv)
        out["gpus"][d] = (busy / 1e6, (span - busy) / 1e6)
    return out


def render_trace_svg(graph, show_dep_arrows: bool = False, out=None) -> str:
    """Timeline SVG: one lane per (GPU, stream) with the tasks' CUDA-event
    intervals, the ready-count curve beneath; prints the idle metric per lane
    and per GPU to ``out`` (stdout by default), like the reference's extension."""
    import sys

    events = graph.trace.export_events()
    lanes = build_lanes(events)
    steps = build_ready_steps(events)
    t_lo = min([e[1] for e in events], default=0)
    t_hi = max([e[1] for e in events], default=1)
    span = max(t_hi - t_lo, 1)
    left, plot_w, lane_h, gap, top, curve_h = 110, 1000, 22, 6, 30, 90
    wids = sorted(lanes)

    def x(t):
        return left + (t - t_lo) / span * plot_w

    def lane_y(i):
        return top + i * (lane_h + gap)

    curve_top = lane_y(max(len(wids), 1)) + 30
    height = curve_top + curve_h + 40
    width = left + plot_w + 30
    parts = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width}" height="{height}" '
             f'viewBox="0 0 {width} {height}">',
             f'<rect x="0" y="0" width="{width}" height="{height}" fill="white"/>']
    pos = {}
    nstreams = graph.engine.worker_stride() if graph.engine else 1
    for i, wid in enumerate(wids):
        y = lane_y(i)
        parts.append(f'<text x="6" y="{y + lane_h * 0.7:.1f}" font-size="11" font-family="sans-serif">'
                     f'gpu{wid // nstreams} s{wid % nstreams}</text>')
        for start, end, tid in lanes[wid]:
            x0, x1 = x(start), x(end)
            w = max(x1 - x0, 0.5)
            parts.append(f'<rect x="{x0:.2f}" y="{y}" width="{w:.2f}" height="{lane_h}" fill="#4c78a8" '
                         f'stroke="#333" stroke-width="0.3"><title>{graph._label(tid)}</title></rect>')
            pos[tid] = (x0, x1, y + lane_h / 2)
    if show_dep_arrows:
        for src, dst, _ in graph.edges():
            if src in pos and dst in pos:
                parts.append(f'<line x1="{pos[src][1]:.2f}" y1="{pos[src][2]:.2f}" x2="{pos[dst][0]:.2f}" '
                             f'y2="{pos[dst][2]:.2f}" stroke="#888" stroke-width="0.6"/>')
    max_count = max([c for _, c in steps], default=1) or 1
    base = curve_top + curve_h
    pts, prev = [], 0
    for t, c in steps:
        xx = x(t) if t else left
        pts.append(f"{xx:.2f},{base - prev / max_count * curve_h:.2f}")
        pts.append(f"{xx:.2f},{base - c / max_count * curve_h:.2f}")
        prev = c
    parts.append(f'<text x="6" y="{curve_top + 12}" font-size="11" font-family="sans-serif">'
                 f'ready tasks (max {max_count})</text>')
    parts.append(f'<polyline points="{" ".join(pts)}" fill="none" stroke="#c44" stroke-width="1.2"/>')
    parts.append("</svg>")
    rep = idle_report(graph, events)
    out = sys.stdout if out is None else out
    for label, (busy, idle) in rep["lanes"].items():
        print(f"[trace] {label}: idle {idle:.3f} ms of {rep['span_ms']:.3f} ms", file=out)
    for d, (busy, idle) in rep["gpus"].items():
        print(f"[trace] gpu{d} (any stream busy): idle {idle:.3f} ms of {rep['span_ms']:.3f} ms "
              f"({100.0 * busy / max(rep['span_ms'], 1e-12):.1f} % busy)", file=out)
    return "\n".join(parts) + "\n"


def generate_trace_svg(graph, path=None, show_dep_arrows: bool = False, out=None) -> str:
    text = render_trace_svg(graph, show_dep_arrows, out)
    if path is not None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
    return text
