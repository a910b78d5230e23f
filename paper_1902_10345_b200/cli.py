"""Command line for the B200 backend: ``python -m paper_1902_10345_b200``.

Mirrors the reference CLI's ``run`` and ``codegen`` subcommands (cli.py:120-
130, :214-238) for on-disk ``.sdfg.json`` graphs (serialization.py:106-160),
with the same exit codes (0 ok, 1 validation, 2 usage, 3 runtime) and
``--format json``:

    run GRAPH [--input TENSORS.json] [--journal J.json] [--precision native|fp32]
              [--stream-order any|fifo]
        marks the program for the GPU (GPUTransformMap's marker), dispatches it
        to a motif kernel or the generic lowering, runs it, and prints an
        ExecutionReport-shaped document (interpreter.py:107-132): outputs
        (value_cap 4096), states_visited, elements_moved of every statically
        countable edge, tasklet_invocations, and the kernel path.
    codegen GRAPH --out DIR [--compile]
        writes the B200 program (the motif binding, or the generated CUDA
        translation unit) plus a build script; --compile builds it.

``--journal`` replays a transformation journal first (engine.py:226-239);
that needs the reference package importable, as journals name its rules.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from typing import Optional

import numpy as np

from . import expr as X
from .dispatch import STORAGE_PREFIX, generate, gpu_storage, invoke_toolchain
from .errors import CodegenError, ExecutionError, ToolchainError
from .generic import compile_generic
from .graph import Graph, GraphFormatError, from_json

EXIT_OK, EXIT_VALIDATION, EXIT_USAGE, EXIT_RUNTIME = 0, 1, 2, 3


class CliError(RuntimeError):
    def __init__(self, message: str, code: int = EXIT_RUNTIME):
        super().__init__(message)
        self.code = code


def _load_doc(path: str) -> dict:
    try:
        with open(path) as f:
            return json.load(f)
    except FileNotFoundError:
        raise CliError(f"no such file: {path}", EXIT_USAGE)
    except json.JSONDecodeError as exc:
        raise CliError(f"cannot load graph from {path}: {exc}")


def _replay(doc: dict, journal_path: str) -> dict:
    try:
        from sdfg.rewriting import replay_journal
        from sdfg.serialization import from_json as ref_from_json, load_journal, to_json
    except ImportError as exc:
        raise CliError(f"--journal needs the reference package (sdfg) importable: {exc}", EXIT_USAGE)
    with open(journal_path) as f:
        jdoc = load_journal(f.read())
    return to_json(replay_journal(ref_from_json(json.dumps(doc)), jdoc["entries"]))


def _mark(doc: dict, precision: str, order: str) -> dict:
    """GPUTransformMap's marker on every non-transient container, unless
    the graph already carries one."""
    data = doc.get("data", [])
    if any((d.get("storage") or "").startswith(STORAGE_PREFIX) for d in data):
        return doc
    doc = json.loads(json.dumps(doc))
    for d in doc["data"]:
        if not d["transient"]:
            d["storage"] = gpu_storage(precision, order)
    return doc


def states_visited(g: Graph, symbols: dict, cap: int = 1_000_000) -> Optional[list]:
    """The state sequence of the interstate machine (interpreter.py:690-710)
    when every condition and assignment depends on symbols only; None when
    control flow reads data (it is then decided on the device)."""
    env = {k: int(v) for k, v in symbols.items()}
    seq, cur = [], g.start_state
    data = set(g.data)
    while cur is not None and len(seq) < cap:
        seq.append(cur)
        nxt = None
        for t in g.out_transitions(cur):
            names = X.free_symbols(t.condition)
            for _, v in t.assignments:
                names |= X.free_symbols(v)
            if names & data:
                return None
            try:
                ok = X.evaluate(t.condition, env)
            except X.ExprError:
                return None
            if ok:
                for k, v in t.assignments:
                    env[k] = X.evaluate(v, env)
                nxt = t.dst
                break
        cur = nxt
    return seq


def _visits(g: Graph, symbols: dict, cap: int = 100_000):
    """(state, symbol env) per visit of the interstate machine, or None when
    control flow reads data (then decided on the device)."""
    env = {k: int(v) for k, v in symbols.items()}
    out, cur = [], g.start_state
    data = set(g.data)
    while cur is not None and len(out) < cap:
        out.append((cur, dict(env)))
        nxt = None
        for t in g.out_transitions(cur):
            names = X.free_symbols(t.condition)
            for _, v in t.assignments:
                names |= X.free_symbols(v)
            if names & data:
                return None
            try:
                ok = X.evaluate(t.condition, env)
            except X.ExprError:
                return None
            if ok:
                for k, v in t.assignments:
                    env[k] = X.evaluate(v, env)
                nxt = t.dst
                break
        cur = nxt
    return out


def _instances(st, parent: dict, scope, env: dict, limit: int = 200_000, per_point=None):
    """Points of the map nest ending at ``scope`` (inclusive ranges,
    symbolic.py:579-618) -- or the sum of ``per_point(env)`` over them;
    None when a range is data-dependent or the nest is too large to
    enumerate."""
    chain = []
    p = scope
    while p is not None:
        chain.append(st.nodes[p])
        p = parent[p]
    chain.reverse()
    for n in chain:
        if n.kind != "map_entry" or any(e.dst_conn and not e.dst_conn.startswith("IN_") and not e.memlet.is_empty
                                        for e in st.in_edges(n.id)):
            return None
    count = 0
    total = 0

    def rec(k, e):
        nonlocal count, total
        if count > limit:
            return
        if k == len(chain):
            count += 1
            total += 1 if per_point is None else per_point(e)
            return
        n = chain[k]

        def dims(d, e2):
            if d == len(n.params):
                rec(k + 1, e2)
                return
            r = n.ranges[d]
            b, en, sd = (int(X.evaluate(x, e2)) for x in (r.begin, r.end, r.stride))
            for v in (range(b, en + 1, sd) if sd > 0 else range(b, en - 1, sd)):
                if count > limit:
                    return
                e3 = dict(e2)
                e3[n.params[d]] = v
                dims(d + 1, e3)
        dims(0, e)
    try:
        rec(0, dict(env))
    except X.ExprError:
        return None
    return None if count > limit else total


def execution_report(g: Graph, symbols: dict) -> dict:
    """The static part of the interpreter's ExecutionReport
    (interpreter.py:107-132): states_visited, elements_moved for every
    memlet edge whose volume is static (accesses x points of its scope x
    visits), and tasklet_invocations when every tasklet's scope can be
    counted.  Dynamic memlets (stream pushes, data-dependent ranges) are
    listed under ``dynamic_edges``: their volumes are data-dependent."""
    visits = _visits(g, symbols)
    if visits is None:
        return {"states_visited": None}
    moved, dynamic = {}, set()
    tasklets = 0
    for name, env in visits:
        st = g.state(name)
        parent = st.scope_parent()
        for e in st.edges:
            key = f"{name}:e{e.id}"
            m = e.memlet
            src = st.nodes[e.src]
            if m.is_empty:
                moved[key] = moved.get(key, 0)
                continue
            if g.data[m.data].kind == "stream" and src.kind == "map_entry":
                moved[key] = moved.get(key, 0)  # stream handles move nothing (interpreter.py:527-530)
                continue
            if m.accesses is None or src.kind in ("consume_entry", "consume_exit"):
                dynamic.add(key)
                continue
            scope = src.id if src.kind == "map_entry" else (
                parent[src.doc["entry"]] if src.kind == "map_exit" else parent[src.id])
            if src.kind == "map_entry":
                # a scope instance reads the memlet's whole block (interpreter.py:531-533)
                def vol(pe, sub=m.subset):
                    v = 1
                    for r in sub:  # points x vector tile (symbolic.py:579-618)
                        b, en, sd = (int(X.evaluate(x, pe)) for x in (r.begin, r.end, r.stride))
                        v *= max(0, (en - b) // sd + 1) * int(X.evaluate(r.tile, pe))
                    return v
                cnt = _instances(st, parent, scope, env, per_point=vol)
            else:
                cnt = _instances(st, parent, scope, env, per_point=lambda pe, a=m.accesses: int(X.evaluate(a, pe)))
            if cnt is None:
                dynamic.add(key)
                continue
            moved[key] = moved.get(key, 0) + cnt
        for n in st.nodes:
            if n.kind == "nested":  # its own edges count under the nested graph's prefix
                dynamic.add(f"{name}:nested{n.id}")
            if tasklets is None:
                continue
            if n.kind in ("nested", "consume_entry"):
                tasklets = None
            elif n.kind == "tasklet":
                pts = _instances(st, parent, parent[n.id], env)
                tasklets = None if pts is None else tasklets + pts
    for k in dynamic:
        moved.pop(k, None)
    rep = {"states_visited": [s for s, _ in visits], "elements_moved": dict(sorted(moved.items())),
           "dynamic_edges": sorted(dynamic), "tasklet_invocations": tasklets}
    if not dynamic:
        rep["total_moved"] = sum(moved.values())
    return rep


def cmd_run(args) -> int:
    doc = _load_doc(args.graph)
    if args.journal:
        doc = _replay(doc, args.journal)
    arrays, symbols = {}, {}
    if args.input:
        with open(args.input) as f:
            t = json.load(f)
        arrays = {k: np.asarray(v) for k, v in t.get("arrays", {}).items()}
        symbols = {k: int(v) for k, v in t.get("symbols", {}).items()}
    marked = _mark(doc, args.precision, args.stream_order)
    g = from_json(marked)
    measured = None
    if args.report == "device":
        # the generic lowering's counter build: every edge measured on the GPU
        prog = compile_generic(from_json(doc), report=True)
        outputs, measured = prog.run_report(arrays, symbols)
        rep = {"outputs": {}, "backend": "b200", "path": "generic", "precision": "native",
               "stream_order": "any", "report": "device"}
    else:
        code = generate(marked)
        prog = invoke_toolchain(code)
        outputs = prog.run(arrays, symbols)
        rep = {"outputs": {}, "backend": "b200",
               "path": f"motif:{code.plan.motif}" if code.plan is not None else "generic",
               "precision": code.precision, "stream_order": code.stream_order, "report": "static"}
    for name, arr in outputs.items():
        shape = [int(X.evaluate(d, symbols)) for d in g.data[name].dims]
        a = np.asarray(arr).reshape(shape)
        rep["outputs"][name] = a.tolist() if a.size <= 4096 else {"truncated": True, "size": int(a.size)}
    if measured is not None:
        rep.update(measured)
    else:
        rep.update({k: v for k, v in execution_report(g, symbols).items() if v is not None})
    print(json.dumps(rep, indent=2, sort_keys=True) if args.format == "json" else json.dumps(rep, sort_keys=True))
    return EXIT_OK


def cmd_codegen(args) -> int:
    doc = _mark(_load_doc(args.graph), args.precision, args.stream_order)
    code = generate(doc)
    os.makedirs(args.out, exist_ok=True)
    generic = code.lowered is not None
    src = os.path.join(args.out, f"{code.name}.cu" if generic else f"{code.name}.b200.txt")
    with open(src, "w") as f:
        f.write(code.source)
    script = os.path.join(args.out, "build.sh")
    with open(script, "w") as f:
        if generic:
            f.write("#!/bin/sh\nset -e\n${NVCC:-nvcc} -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 "
                    f"-fmad=false --expt-relaxed-constexpr -Xcompiler -fPIC -shared {code.name}.cu "
                    f"-o lib{code.name}.so -lcudart\n")
        else:
            f.write("#!/bin/sh\n# motif kernels live in the prebuilt libsdfgb200.so\n"
                    "make -C \"$(dirname \"$0\")\"/../paper_1902_10345_b200/csrc\n")
    os.chmod(script, 0o755)
    compiled = None
    if args.compile:
        compiled = invoke_toolchain(code).path if generic else "libsdfgb200.so (prebuilt)"
    payload = {"source": src, "build_script": script, "compiled": compiled,
               "path": "generic" if generic else f"motif:{code.plan.motif}"}
    print(json.dumps(payload, indent=2, sort_keys=True) if args.format == "json" else f"wrote {src}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_1902_10345_b200",
                                description="Run and compile SDFG graphs on a B200 (sm_100a).")
    p.add_argument("--format", choices=("text", "json"), default="text")
    sub = p.add_subparsers(dest="command", required=True)
    for name, fn, hlp in (("run", cmd_run, "execute a graph on the GPU"),
                          ("codegen", cmd_codegen, "emit the B200 program")):
        s = sub.add_parser(name, help=hlp)
        s.add_argument("graph")
        s.add_argument("--precision", choices=("fp32", "native"), default="native")
        s.add_argument("--stream-order", choices=("any", "fifo"), default="any")
        if name == "run":
            s.add_argument("--input", help="JSON tensor file with arrays and symbols")
            s.add_argument("--journal", help="transformation journal to replay first")
            s.add_argument("--report", choices=("static", "device"), default="static",
                           help="ExecutionReport: static volumes (dynamic edges listed), or every edge "
                                "counted on the device by the generic lowering's counter build")
        else:
            s.add_argument("--out", required=True)
            s.add_argument("--compile", action="store_true")
        s.set_defaults(fn=fn)
    return p


def main(argv: Optional[list] = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        return args.fn(args)
    except CliError as exc:
        code, msg = exc.code, str(exc)
    except (CodegenError, GraphFormatError) as exc:
        code, msg = EXIT_VALIDATION, f"{type(exc).__name__}: {exc}"
    except (ExecutionError, ToolchainError, Exception) as exc:  # runtime failures stay machine-readable
        code, msg = EXIT_RUNTIME, f"{type(exc).__name__}: {exc}"
    if args.format == "json":
        print(json.dumps({"error": msg}))
    else:
        print(f"error: {msg}", file=sys.stderr)
    return code
