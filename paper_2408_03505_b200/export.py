"""Schedule export: the chosen candidate's schedule as a
JSON document or a Chrome trace (chrome://tracing, Perfetto), the hand-off the
paper's runtime reads as "schedule configuration files".

Formatting only: every time and placement comes from the library's GPU
results (optimus_explain, optimus_emit_schedule, optimus_emit_p2p,
optimus_debug_template).  Times are LLM-relative (template) nanoseconds; the
executed iteration runs the LLM Df later (R10) and adds Db at its end (R16).
"""
from __future__ import annotations

import json


def _llm_busy(free, w, z):
    """Busy blocks of one LLM resource on one stage: [w, z] minus its free intervals."""
    out, t = [], w
    for lo, hi in sorted(free):
        if lo > t:
            out.append((t, lo))
        t = max(t, hi)
    if t < z:
        out.append((t, z))
    return out


def schedule(ctx, g: int, stream=None) -> dict:
    """JSON-ready schedule of candidate g."""
    x = ctx.explain(g, stream=stream)
    em = ctx.emit_schedule(g, stream=stream)
    p2p = ctx.emit_p2p(g, stream=stream)
    tpl = ctx.debug_template(stream=stream)
    plan = ctx.get_plan(x["plan"])
    return {
        "candidate": int(g), "lat_ns": x["lat"], "delta_f_ns": x["df"], "delta_b_ns": x["db"],
        "T_end_ns": tpl["T_end"], "encoder_plan": {"dp": plan["dp"], "pp": plan["pp"], "tp": plan["tp"], "m": plan["m"]},
        "partition": x["N"], "coarse_forward": x["c_final"], "coarse_backward": x["cb_final"],
        "forward_moves": x["moves_f"], "backward_moves": x["moves_b"],
        "encoder_kernels": {"fields": ["pipeline", "stage", "comm", "start_ns", "end_ns", "move"],
                            "forward": em["fwd_place"], "backward": em["bwd_place"]},
        "p2p": {"fields": ["dir", "microbatch", "pipeline", "src_stage", "src_slot", "dst_stage", "dst_slot",
                           "send_ns", "arrive_ns"], "records": p2p},
        "llm": {"warmup": tpl["W"], "F_ns": tpl["F"], "B_ns": tpl["B"], "w_ns": tpl["w"], "z_ns": tpl["z"],
                "compute_busy": [_llm_busy(tpl["comp_free"][s], tpl["w"][s], tpl["z"][s]) for s in range(len(tpl["w"]))],
                "comm_free": tpl["comm_free"]},
        "time_base": "LLM-relative (template) ns; executed LLM = template + delta_f",
    }


def chrome_trace(ctx, g: int, stream=None) -> dict:
    """Chrome trace events: pid = LLM stage (device row of one LLM pipeline),
    tid 0 LLM compute, tid 1 + pipeline encoder kernels, tid 100 P2P; us."""
    sch = schedule(ctx, g, stream=stream)
    ev = []
    us = lambda ns: ns / 1000.0  # noqa: E731
    for s, blocks in enumerate(sch["llm"]["compute_busy"]):
        for lo, hi in blocks:
            ev.append({"name": "LLM compute", "ph": "X", "pid": s, "tid": 0, "ts": us(lo), "dur": us(hi - lo)})
    plan = sch["encoder_plan"]
    rt = max(1, plan["m"] // max(1, len(sch["llm"]["w_ns"]) // plan["pp"]))
    for key in ("forward", "backward"):
        for pj, st, comm, lo, hi, mv in sch["encoder_kernels"][key]:
            stage = (pj // rt) * plan["pp"] + st
            ev.append({"name": f"enc {key} {'comm' if comm else 'compute'} (pipeline {pj}, move {mv})", "ph": "X",
                       "pid": stage, "tid": 1 + pj, "ts": us(lo), "dur": us(hi - lo)})
    for d, i, pj, ss, sb, ds, db, t0, t1 in sch["p2p"]["records"]:
        nm = f"p2p {'activation' if d == 0 else 'gradient'} mb {i} (pipeline {pj})"
        ev.append({"name": nm + " send", "ph": "X", "pid": ss, "tid": 100, "ts": us(t0), "dur": us(t1 - t0)})
        ev.append({"name": nm + " recv", "ph": "X", "pid": ds, "tid": 100, "ts": us(t0), "dur": us(t1 - t0)})
    return {"traceEvents": ev, "displayTimeUnit": "ns",
            "otherData": {k: v for k, v in sch.items() if k in ("candidate", "lat_ns", "delta_f_ns", "delta_b_ns",
                                                                 "T_end_ns", "encoder_plan", "partition", "time_base")}}


def write(ctx, g: int, path: str, fmt: str = "chrome", stream=None) -> None:
    doc = chrome_trace(ctx, g, stream) if fmt == "chrome" else schedule(ctx, g, stream)
    with open(path, "w") as f:
        json.dump(doc, f)
