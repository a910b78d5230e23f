"""Host-side logic (no GPU): expression handling, motif classification,
GPUTransformMap in the reference's rewriting engine, the drop-in's error
behaviour, and the C ABI surface of libsdfgb200.so."""

import ctypes
import json
import os
import sys

import numpy as np
import pytest

from conftest import REPO, graph_path, load_cases, reference_available

import paper_1902_10345_b200 as b200
from paper_1902_10345_b200 import _lib, expr as X
from paper_1902_10345_b200.classify import UnsupportedGraph, classify, match_histogram
from paper_1902_10345_b200.graph import load

needs_ref = pytest.mark.skipif(not reference_available(), reason="reference not mounted")


# ------------------------------------------------------------------ C ABI

def test_library_exports_every_declared_symbol():
    L = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} lacks a ctypes signature"
    assert L.sdfgb_abi_version() == 1


def test_workspace_queries_need_no_gpu():
    L = _lib.load()
    assert L.sdfgb_query_workspace_bytes(1 << 26, 4) >= (1 << 26) // 16384 * 8
    assert L.sdfgb_gemm_workspace_bytes(128, 256, 64) == 2 * 128 * 64 * 4 + 2 * 256 * 64 * 4


def test_invalid_arguments_are_rejected_before_any_launch():
    L = _lib.load()
    rc = L.sdfgb_hist_f32(None, -1, 256.0, 1.0, None, 256, None, None)
    assert rc == _lib.ERR_INVALID
    assert b"hist" in L.sdfgb_last_error()
    with pytest.raises(b200.CodegenError):
        _lib.check(rc)


def test_sass_is_sm100a_tcgen05():
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out or "UTCQMMA" in out, "no tcgen05 MMA in the GEMM"
    assert "UTMALDG" in out, "no TMA loads"
    assert "LDTM" in out, "no TMEM loads"
    elf = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in elf


# ------------------------------------------------------------- expressions

def test_expression_floor_semantics_match_reference_helpers():
    # sdfg_fdiv / sdfg_fmod (tasklets.py:336-347): floor semantics
    assert X.evaluate(X.parse_expr("-7 // 2"), {}) == -4
    assert X.evaluate(X.parse_expr("-7 % 2"), {}) == 1
    assert X.evaluate(X.parse_expr("(t + 1) % 2"), {"t": 3}) == 0
    assert X.evaluate(X.parse_expr("min(N - 1, i_t + 3)"), {"N": 10, "i_t": 8}) == 9


def test_ranges_and_subsets():
    r = X.parse_range("0:M - 1:4")
    assert X.evaluate(r.stride, {}) == 4 and X.evaluate(r.end, {"M": 9}) == 8
    s = X.parse_subset("[t % 2, i - 1, min(N - 1, j + 3)]")
    assert len(s) == 3 and s[0].is_point
    a = X.affine(X.parse_expr("(k - k_t) + k_t"))
    assert a.only("k") == 0
    assert X.affine(X.parse_expr("i * 2 + j")).terms == {"i": 2, "j": 1}


# ---------------------------------------------------------- classification

EXPECT = {
    "histogram": ("histogram", {"img": "img", "hist": "hist"}),
    "histogram_int": ("histogram_int", {"img": "img", "hist": "hist"}),
    "query": ("query", {"col": "col", "thr": "thr", "out_vals": "out_vals", "count": "count"}),
    "query_gallery": ("query", {"col": "col", "thr": "thr", "out_vals": "out_vals", "count": "count"}),
    "spmv": ("spmv", {"rowptr": "A_row", "col": "A_col", "val": "A_val", "x": "x", "b": "b"}),
    "jacobi2d": ("jacobi2d", {"A": "A"}),
    "matmul": ("matmul", {"A": "A", "B": "B", "C": "C"}),
    "matmul_raw": ("matmul", {"A": "A", "B": "B", "C": "C"}),
    "matmul_tiled": ("matmul", {"A": "A", "B": "B", "C": "C"}),
    "matmul_chain": ("matmul", {"A": "A", "B": "B", "C": "C"}),
}


@pytest.mark.parametrize("name", sorted(EXPECT))
def test_golden_graphs_classify(name):
    plan = classify(load(graph_path(name)))
    motif, roles = EXPECT[name]
    assert plan.motif == motif
    assert plan.roles == roles


def test_classified_parameters():
    h = classify(load(graph_path("histogram")))
    assert (h.params["scale"], h.params["div"], str(h.params["bins"])) == (256.0, 1.0, "256")
    q = classify(load(graph_path("query")))
    assert q.params["op"] == "<"
    assert classify(load(graph_path("query_gallery"))).params["op"] == ">"
    j = classify(load(graph_path("jacobi2d")))
    assert j.params["coef"] == 0.2
    assert j.params["terms"] == [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)]
    assert str(j.params["steps"]) == "T" and str(j.params["N"]) == "N"
    s = classify(load(graph_path("spmv")))
    assert s.pointer_args[0] == ("A_row", "int64") and s.symbol_args == ["H", "W", "nnz"]


@pytest.mark.parametrize("name", ["histogram_looped", "query_cond"])
def test_motif_under_control_flow_is_not_a_motif(name):
    """A motif state in a guard loop or behind a condition may run zero or
    several times; the motif kernel runs it once, so the classifier must
    refuse it and the generic lowering (a state machine) runs it."""
    with pytest.raises(UnsupportedGraph, match="control flow|conditional|revisits|assigns"):
        classify(load(graph_path(name)))
    doc = json.load(open(graph_path(name)))
    for d in doc["data"]:
        if not d["transient"]:
            d["storage"] = "GPU_Global:native"
    code = b200.generate(doc)
    assert code.plan is None and code.lowered is not None


def test_histogram_with_extra_body_tasklet_is_not_a_motif():
    doc = json.load(open(graph_path("histogram")))
    st = doc["states"][0]
    extra = json.loads(json.dumps([n for n in st["nodes"] if n["kind"] == "tasklet" and n["name"] == "binner"][0]))
    extra["name"] = "spare"
    st["nodes"].append(extra)
    me = [i for i, n in enumerate(st["nodes"]) if n["kind"] == "map_entry"][0]
    st["edges"].append({"src": me, "src_conn": None, "dst": len(st["nodes"]) - 1, "dst_conn": None,
                        "memlet": {"empty": True}})
    with pytest.raises(UnsupportedGraph, match="besides the binner"):
        match_histogram(load(doc))


def test_non_motif_programs_take_the_generic_lowering():
    with pytest.raises(UnsupportedGraph):
        classify(load(graph_path("laplace1d")))  # 1-D 'l - 2*c + r' stencil: no motif kernel
    code = b200.generate(graph_path("laplace1d"), require_marked=False)
    assert code.plan is None and code.lowered is not None
    doc = json.load(open(graph_path("gal_fibonacci")))
    for st in doc["states"]:
        for n in st["nodes"]:
            if n["kind"] == "consume_entry":
                n["condition"] = "size(S) > 3"  # not a drain-until-empty consume: not lowerable
    with pytest.raises(b200.CodegenError):
        b200.generate(doc, require_marked=False)


def test_mutated_programs_are_rejected():
    doc = json.load(open(graph_path("histogram")))
    # WCR max instead of sum on the subscript write
    for st in doc["states"]:
        for e in st["edges"]:
            if e["memlet"].get("wcr"):
                e["memlet"]["wcr"]["kind"] = "max"
    with pytest.raises(UnsupportedGraph):
        classify(load(doc))
    doc = json.load(open(graph_path("jacobi2d")))
    for st in doc["states"]:
        for n in st["nodes"]:
            if n["kind"] == "tasklet":
                n["code"] = "o = 0.2 * (c + (n + s) + w + e)"  # different summation order
    with pytest.raises(UnsupportedGraph):
        classify(load(doc))


def test_generate_requires_the_transformation():
    with pytest.raises(b200.CodegenError, match="GPUTransformMap"):
        b200.generate(graph_path("query"))


def test_generated_signature_matches_reference_order():
    code = b200.generate(graph_path("spmv"), require_marked=False)
    assert code.signature() == ("void spmv(int64_t* A_row, int64_t* A_col, double* A_val, double* x, "
                                "double* b, int64_t H, int64_t W, int64_t nnz)")
    assert "sdfgb_host_spmv" in code.source


def test_run_rejects_bad_inputs():
    prog = b200.compile_b200(graph_path("query"))
    with pytest.raises(b200.ExecutionError, match="unbound"):
        prog.run({}, {})
    with pytest.raises(b200.ExecutionError, match="elements"):
        prog.run({"col": np.zeros(3), "thr": [0.5], "out_vals": np.zeros(4), "count": [0]}, {"N": 4})


# ------------------------------------------------- reference integration

@needs_ref
class TestGPUTransformMapInReference:
    @pytest.fixture(autouse=True)
    def _registered(self):
        sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
        import motifs_ref  # noqa: F401  (puts the reference on sys.path)
        from sdfg import rewriting
        b200.register(rewriting)
        yield
        b200.unregister(rewriting)

    def _builders(self):
        import motifs_ref as M
        return {"histogram": M.histogram, "query": M.query, "spmv": M.spmv, "jacobi2d": M.jacobi2d,
                "matmul": M.matmul, "matmul_chain": M.BUILDERS["matmul_chain"],
                "histogram_int": M.histogram_int}

    def test_exactly_one_match_per_motif(self):
        from sdfg.rewriting import find_matches
        for name, build in self._builders().items():
            ms = find_matches(build(), "GPUTransformMap")
            assert len(ms) == 1, name

    def test_apply_marks_storage_and_journals_precision(self):
        from sdfg.rewriting import apply_transformation, find_matches
        g = self._builders()["query"]()
        g2, entry = apply_transformation(g, find_matches(g, "GPUTransformMap")[0], {"precision": "fp32"})
        assert entry["transformation"] == "GPUTransformMap"
        assert entry["params"] == {"precision": "fp32"}  # non-default parameters are journaled
        assert g2.data["col"].storage == "GPU_Global:fp32"
        assert g.data["col"].storage == "heap"  # input graph untouched (engine.py:195)
        assert find_matches(g2, "GPUTransformMap") == []  # not re-applicable
        code = b200.generate(g2)
        assert code.precision == "fp32" and code.plan.motif == "query"

    def test_marked_graph_stays_valid_for_the_interpreter(self):
        from sdfg.interpreter import run
        from sdfg.rewriting import apply_transformation, find_matches
        from sdfg.validation import validate_sdfg
        g = self._builders()["histogram"]()
        g2, _ = apply_transformation(g, find_matches(g, "GPUTransformMap")[0])
        assert [d for d in validate_sdfg(g2) if d.severity == "error"] == []
        img = np.random.default_rng(0).random((5, 6))
        a = run(g, {"img": img, "hist": np.zeros(256, np.int64)}, {"H": 5, "W": 6}).outputs["hist"]
        b = run(g2, {"img": img, "hist": np.zeros(256, np.int64)}, {"H": 5, "W": 6}).outputs["hist"]
        assert np.array_equal(a, b)

    def test_journal_replays(self):
        from sdfg.rewriting import apply_transformation, find_matches, replay_journal
        g = self._builders()["jacobi2d"]()
        g2, entry = apply_transformation(g, find_matches(g, "GPUTransformMap")[0])
        g3 = replay_journal(g, [entry])
        assert g3.data["A"].storage == g2.data["A"].storage == "GPU_Global:native"

    def test_hot_path_transformations_keep_the_motif(self):
        """a9: MapTiling / LocalStorage / MapExpansion keep the classification."""
        from sdfg.rewriting import apply_transformation, find_matches
        for name, build in self._builders().items():
            if name == "matmul_chain":
                continue  # already tiled; re-tiling shadows 'i_t' (library.py:576-580)
            base = classify(load(build()))
            g = build()
            for rule in ("MapTiling", "MapExpansion"):
                ms = [m for m in find_matches(g, rule) if m.state == base.main_state]
                if ms:
                    g, _ = apply_transformation(g, ms[0])
            plan = classify(load(g))
            assert plan.motif == base.motif and plan.roles == base.roles, name
            assert len(find_matches(g, "GPUTransformMap")) == 1, name


def test_missing_native_library_fails_loudly(tmp_path, monkeypatch):
    """no CPU fallback: without libsdfgb200.so the product path raises"""
    from paper_1902_10345_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.BackendUnavailable, match="not built"):
        _lib.load(str(tmp_path / "libsdfgb200.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "libsdfgb200.so"))
    import paper_1902_10345_b200 as b200
    doc = json.load(open(graph_path("histogram")))
    for d in doc["data"]:
        if not d["transient"]:
            d["storage"] = "GPU_Global:fp32"
    with pytest.raises(Exception) as ei:
        b200.invoke_toolchain(b200.generate(doc))
    assert "libsdfgb200" in str(ei.value) or "not built" in str(ei.value)


# ------------------------------------------- the reference's own toolchain

@needs_ref
@pytest.mark.parametrize("name", ["histogram", "query", "spmv", "jacobi2d", "matmul"])
def test_reference_toolchain_builds_and_calls_the_shim(name, tmp_path):
    """The reference's UNMODIFIED invoke_toolchain + CompiledSdfg (codegen.py:
    866-913) take the B200 GeneratedB200Code as they take their own: cc
    compiles its source, ctypes binds ``getattr(lib, code.name)`` and
    ``run`` calls it with (*ptrs, *int64 syms).  Without a device the entry
    reports SDFGB_ERR_CUDA through sdfgb_last_status() instead of crashing."""
    sys.path.insert(0, "/root/reference/pkg/src")
    from sdfg import codegen as ref_codegen
    code = b200.generate(graph_path(name), require_marked=False)
    prog = ref_codegen.invoke_toolchain(code, flags=b200.dispatch.shim_link_flags(), workdir=str(tmp_path))
    case = load_cases(name)[0]
    prog.run(case.inputs, case.symbols)
    L = _lib.load()
    status = L.sdfgb_last_status()
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:
        have_gpu = False
    if not have_gpu:
        assert status == _lib.ERR_CUDA
        assert b"CUDA" in L.sdfgb_last_error() or b"cuda" in L.sdfgb_last_error()


def test_shim_source_has_the_reference_signature():
    for name in ("histogram", "query", "spmv", "jacobi2d", "matmul", "histogram_int"):
        code = b200.generate(graph_path(name), require_marked=False)
        assert code.signature() + " {" in code.source
        assert "sdfgb_host_" in code.source
