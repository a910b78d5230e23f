"""CLI (paper_1902_10345_b200/cli.py): the reference CLI's run/codegen shape
for on-disk graphs.  CPU tests cover parsing, marking, codegen and the
interstate simulation; the GPU test runs a graph end to end."""

import json
import os

import numpy as np
import pytest

from conftest import graph_path, load_cases

from paper_1902_10345_b200 import cli
from paper_1902_10345_b200.graph import load


def test_states_visited_follows_the_guard_loop():
    g = load(graph_path("jacobi2d"))
    sv = cli.states_visited(g, {"N": 6, "T": 3})
    assert sv[0] == g.start_state and len(sv) >= 2 + 2 * 3


def test_states_visited_is_none_for_data_dependent_control_flow():
    assert cli.states_visited(load(graph_path("gal_branching")), {}) is None


def test_codegen_writes_cuda_for_generic_graphs(tmp_path):
    rc = cli.main(["--format", "json", "codegen", graph_path("gal_mandelbrot"), "--out", str(tmp_path)])
    assert rc == 0
    cu = [f for f in os.listdir(tmp_path) if f.endswith(".cu")]
    assert cu and "__global__" in open(tmp_path / cu[0]).read()
    assert os.access(tmp_path / "build.sh", os.X_OK)


def test_codegen_describes_motif_bindings(tmp_path):
    assert cli.main(["codegen", graph_path("histogram"), "--out", str(tmp_path)]) == 0
    txt = [f for f in os.listdir(tmp_path) if f.endswith(".b200.txt")]
    assert txt and "sdfgb_host_histogram" in open(tmp_path / txt[0]).read()


def test_usage_errors_exit_2(tmp_path, capsys):
    assert cli.main(["run", str(tmp_path / "missing.sdfg.json")]) == 2


@pytest.mark.gpu
def test_run_end_to_end(tmp_path, capsys, cuda_ok):
    case = [c for c in load_cases("gal_laplace") if c.case == "seed0"][0]
    inp = tmp_path / "in.json"
    inp.write_text(json.dumps({"arrays": {k: v.tolist() for k, v in case.inputs.items()},
                               "symbols": case.symbols}))
    assert cli.main(["--format", "json", "run", graph_path("gal_laplace"), "--input", str(inp)]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["path"] == "generic"
    np.testing.assert_array_equal(np.array(rep["outputs"]["A"]), case.outputs["A"].reshape(2, -1))
    assert rep["states_visited"][0] == "init"


def test_states_visited_matches_the_reference_interpreter():
    """interstate simulation == interpreter's states_visited on every golden
    case whose control flow reads symbols only"""
    n = 0
    for c in load_cases():
        if c.states is None or c.error:
            continue
        name = c.motif
        sv = cli.states_visited(load(graph_path(name)), c.symbols)
        if sv is None:
            continue
        assert sv == c.states, repr(c)
        n += 1
    assert n > 20


def test_execution_report_matches_the_interpreter_on_static_edges():
    """elements_moved of every statically countable edge and
    tasklet_invocations == the reference interpreter's ExecutionReport"""
    edges = cases = tl = 0
    for c in load_cases():
        if c.moved is None or c.error:
            continue
        rep = cli.execution_report(load(graph_path(c.motif)), c.symbols)
        if rep.get("states_visited") is None:
            continue
        for k, v in rep["elements_moved"].items():
            assert c.moved.get(k, 0) == v, f"{c}: {k}"
            edges += 1
        if not rep["dynamic_edges"]:
            assert rep["total_moved"] == sum(c.moved.values()), repr(c)
        if rep["tasklet_invocations"] is not None:
            assert rep["tasklet_invocations"] == c.tasklets, repr(c)
            tl += 1
        cases += 1
    assert cases > 40 and edges > 400 and tl > 20, (cases, edges, tl)


def _report_cases():
    from paper_1902_10345_b200.lower import LoweringError, lower
    seen = {}
    for c in load_cases():
        if c.moved is None or c.error:
            continue
        if c.motif not in seen:
            try:
                lower(load(graph_path(c.motif)), report=True)
                seen[c.motif] = True
            except LoweringError:
                seen[c.motif] = False
        if seen[c.motif]:
            yield c


def test_report_build_has_a_counter_for_every_counted_edge():
    """the counter build covers every edge key the interpreter reports"""
    from paper_1902_10345_b200.lower import lower
    n = 0
    for c in _report_cases():
        keys = set(lower(load(graph_path(c.motif)), report=True).report_keys)
        missing = [k for k, v in c.moved.items() if v and k not in keys]
        assert not missing, f"{c}: {missing}"
        n += 1
    assert n > 50


@pytest.mark.gpu
def test_device_report_matches_the_interpreter(cuda_ok):
    """ExecutionReport measured on the device (lower(report=True)) ==
    the reference interpreter's, edge by edge, on every golden case --
    including the dynamic edges the static report cannot count (stream
    pushes, data-dependent ranges, consume scopes, nested graphs)"""
    from paper_1902_10345_b200.generic import compile_generic
    progs, n, dyn = {}, 0, 0
    for c in _report_cases():
        if c.motif not in progs:
            progs[c.motif] = compile_generic(load(graph_path(c.motif)), report=True)
        _, rep = progs[c.motif].run_report(c.inputs, c.symbols)
        if c.states is not None:
            assert rep["states_visited"] == c.states, repr(c)
        keys = set(rep["elements_moved"]) | set(c.moved)
        bad = {k: (rep["elements_moved"].get(k, 0), c.moved.get(k, 0)) for k in keys
               if rep["elements_moved"].get(k, 0) != c.moved.get(k, 0)}
        assert not bad, f"{c}: (device, interpreter) {bad}"
        assert rep["total_moved"] == sum(c.moved.values()), repr(c)
        assert rep["tasklet_invocations"] == c.tasklets, repr(c)
        static = cli.execution_report(load(graph_path(c.motif)), c.symbols)
        dyn += bool(static.get("dynamic_edges"))
        n += 1
    assert n > 60 and dyn > 20, (n, dyn)


@pytest.mark.gpu
def test_run_with_device_report(tmp_path, capsys, cuda_ok):
    case = load_cases("spmv")[0]
    inp = tmp_path / "in.json"
    inp.write_text(json.dumps({"arrays": {k: v.tolist() for k, v in case.inputs.items()},
                               "symbols": case.symbols}))
    assert cli.main(["--format", "json", "run", graph_path("spmv"), "--input", str(inp), "--report", "device"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["report"] == "device" and rep["elements_moved"] == {k: v for k, v in sorted(case.moved.items())
                                                                   if k in rep["elements_moved"]}
    assert rep["total_moved"] == sum(case.moved.values())
