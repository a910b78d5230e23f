"""Drop-in execution of GPU-marked SDFGs: the B200 twin of the reference's
``generate`` / ``invoke_toolchain`` / ``CompiledSdfg.run`` (codegen.py:802-913).

    code = generate(sdfg)                 # classify, bind to a kernel family
    prog = invoke_toolchain(code)         # load libsdfgb200.so (prebuilt)
    out  = prog.run(arrays, symbols)      # same contract as CompiledSdfg.run

``run`` mirrors ``CompiledSdfg.run`` (codegen.py:875-887): every
non-transient array is copied into a contiguous buffer of its declared
basetype, the library entry is called with host pointers, and the buffers
are returned (callers reshape as they would for the reference).  The C entry
stages to HBM, runs the sm_100a kernels and copies back; nothing runs on
the CPU.  Errors use the reference's exception names (errors.py).
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from typing import Any, Mapping, Optional

import numpy as np

from . import _lib
from . import expr as X
from .classify import Plan, UnsupportedGraph, classify
from .errors import CodegenError, ExecutionError, ToolchainError
from .graph import Graph, load

STORAGE_PREFIX = "GPU_Global"
PRECISIONS = ("fp32", "native")
_CT = {"int64": "int64_t", "float64": "double"}


STREAM_ORDERS = ("any", "fifo")


def gpu_storage(precision: str, stream_order: str = "any") -> str:
    """The marker GPUTransformMap writes into DataDesc.storage:
    ``GPU_Global:<precision>[:fifo]``."""
    return f"{STORAGE_PREFIX}:{precision}" + (":fifo" if stream_order == "fifo" else "")


def _parse_storage(st: str):
    parts = st.split(":")
    prec = parts[1] if len(parts) > 1 else "fp32"
    order = parts[2] if len(parts) > 2 else "any"
    return prec, order


def marked_mode(g: Graph, plan: Plan) -> Optional[tuple]:
    """(precision, stream_order) recorded by GPUTransformMap on the motif's
    containers (DataDesc.storage is a free string, ir.py:75); None if the
    graph is not marked."""
    seen = set()
    for c in plan.roles.values():
        st = g.data[c].storage or ""
        if st.startswith(STORAGE_PREFIX):
            seen.add(_parse_storage(st))
        else:
            return None
    if len(seen) != 1:
        raise CodegenError(f"inconsistent GPU storage markers {sorted(seen)}")
    return seen.pop()


def marked_precision(g: Graph, plan: Plan) -> Optional[str]:
    mode = marked_mode(g, plan)
    return None if mode is None else mode[0]


@dataclass
class GeneratedB200Code:
    """Counterpart of ``GeneratedCode`` (codegen.py:146-156).  ``plan`` is
    the motif binding; graphs outside the five motifs carry ``lowered``
    (the generic Map/tasklet -> CUDA translation unit, lower.py) instead."""
    source: str
    name: str
    pointer_args: list
    symbol_args: list
    plan: Optional[Plan]
    precision: str
    stream_order: str = "any"
    lowered: Any = None
    graph: Any = None

    def signature(self) -> str:
        parts = [f"{_CT[t]}* {n}" for n, t in self.pointer_args]
        parts += [f"int64_t {s}" for s in self.symbol_args]
        return f"void {self.name}({', '.join(parts)})"


_ENTRY = {
    "histogram": "sdfgb_host_histogram",
    "histogram_int": "sdfgb_host_histogram_i64",
    "query": "sdfgb_host_query",
    "spmv": "sdfgb_host_spmv",
    "jacobi2d": "sdfgb_host_jacobi2d",
    "matmul": "sdfgb_host_matmul",
}


def _describe(plan: Plan, precision: str) -> str:
    params = {k: (str(v) if isinstance(v, X.Expr) else v) for k, v in plan.params.items()}
    return (f"/* {plan.name}: motif '{plan.motif}' -> libsdfgb200.so:{_ENTRY[plan.motif]}\n"
            f" * roles {json.dumps(plan.roles, sort_keys=True)}\n"
            f" * params {json.dumps(params, sort_keys=True)}\n"
            f" * precision {precision}; state '{plan.main_state}', map node {plan.main_map} */\n")


def generate(sdfg: Any, require_marked: bool = True) -> GeneratedB200Code:
    """Classify a (GPUTransformMap-marked) SDFG and bind it to a kernel.

    Raises CodegenError when the graph is not marked or matches no motif --
    the reference raises CodegenError for graphs it cannot emit
    (codegen.py:804-807)."""
    g = load(sdfg)
    try:
        plan = classify(g)
    except UnsupportedGraph as exc:
        return _generate_generic(g, require_marked, exc)
    mode = marked_mode(g, plan)
    if mode is None:
        if require_marked:
            raise CodegenError(
                f"SDFG '{g.name}' has no state matched by GPUTransformMap; apply the "
                f"transformation before generating B200 code")
        mode = ("fp32", "any")
    prec, order = mode
    if prec not in PRECISIONS:
        raise CodegenError(f"unknown precision '{prec}'")
    if order not in STREAM_ORDERS:
        raise CodegenError(f"unknown stream order '{order}'")
    return GeneratedB200Code(_describe(plan, prec), g.name, plan.pointer_args, plan.symbol_args,
                             plan, prec, order)


def generic_marked(g: Graph) -> Optional[tuple]:
    """(precision, stream_order) from the non-transient containers of a
    graph outside the motifs; None when any of them is unmarked."""
    seen = set()
    for d in g.data.values():
        if d.transient:
            continue
        st = d.storage or ""
        if not st.startswith(STORAGE_PREFIX):
            return None
        seen.add(_parse_storage(st))
    if len(seen) > 1:
        raise CodegenError(f"inconsistent GPU storage markers {sorted(seen)}")
    return seen.pop() if seen else None


def _generate_generic(g: Graph, require_marked: bool, why: Exception) -> GeneratedB200Code:
    """Graphs that are none of the five motifs go through the generic
    Map/tasklet lowering (lower.py).  It computes in the
    reference's basetypes (float64/int64) whatever precision was marked."""
    from .lower import LoweringError, lower
    mode = generic_marked(g)
    if mode is None and require_marked:
        raise CodegenError(
            f"SDFG '{g.name}' has no state matched by GPUTransformMap; apply the "
            f"transformation before generating B200 code")
    try:
        lw = lower(g)
    except LoweringError as exc:
        raise CodegenError(f"SDFG '{g.name}': not a motif ({why}) and not lowerable: {exc}") from exc
    order = mode[1] if mode else "any"
    return GeneratedB200Code(lw.source, g.name, lw.pointer_args, lw.symbol_args, None, "native", order,
                             lowered=lw, graph=g)


def invoke_toolchain(code: GeneratedB200Code) -> "CompiledB200Sdfg":
    """Load the prebuilt sm_100a library (the reference compiles with cc
    here, codegen.py:890-913; our kernels are built once by build()).
    Generic programs are compiled with nvcc for sm_100a (generic.py)."""
    if code.lowered is not None:
        from .generic import GenericProgram, build
        return GenericProgram(code.graph, code.lowered, build(code.lowered))
    try:
        lib = _lib.load()
    except _lib.BackendUnavailable as exc:
        raise ToolchainError(str(exc)) from exc
    return CompiledB200Sdfg(code, lib)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class CompiledB200Sdfg:
    """A loaded B200 program; ``run`` has CompiledSdfg.run's contract."""

    def __init__(self, code: GeneratedB200Code, lib):
        self.code = code
        self._lib = lib

    def run(self, arrays: Mapping[str, Any], symbols: Mapping[str, int]) -> dict:
        plan = self.code.plan
        syms = {k: int(v) for k, v in symbols.items()}
        missing = [s for s in plan.symbol_args if s not in syms]
        if missing:
            raise ExecutionError(f"unbound symbols: {sorted(missing)}")
        bufs = {}
        for name, bt in plan.pointer_args:
            if name not in arrays:
                raise ExecutionError(f"missing input container '{name}'")
            dt = np.int64 if bt == "int64" else np.float64
            buf = np.ascontiguousarray(np.asarray(arrays[name], dtype=dt)).copy()
            want = int(np.prod(plan.shape(name, syms)))
            if buf.size != want:
                raise ExecutionError(f"input '{name}' has {buf.size} elements; container expects {want}")
            bufs[name] = buf
        prec = _lib.PREC_FP32 if self.code.precision == "fp32" else _lib.PREC_NATIVE
        getattr(self, "_run_" + plan.motif)(plan, bufs, syms, prec)
        return bufs

    # -- per-motif host entries -------------------------------------------

    def _run_histogram(self, plan, b, syms, prec):
        img, hist = b[plan.roles["img"]], b[plan.roles["hist"]]
        shp = plan.shape(plan.roles["img"], syms)
        H = shp[0]
        W = int(np.prod(shp[1:])) if len(shp) > 1 else 1
        _lib.check(self._lib.sdfgb_host_histogram(_ptr(img), _ptr(hist), H, W, hist.size,
                                                  plan.params["scale"], plan.params["div"], prec))

    def _run_histogram_int(self, plan, b, syms, prec):
        img, hist = b[plan.roles["img"]], b[plan.roles["hist"]]
        shp = plan.shape(plan.roles["img"], syms)
        H = shp[0]
        W = int(np.prod(shp[1:])) if len(shp) > 1 else 1
        _lib.check(self._lib.sdfgb_host_histogram_i64(_ptr(img), _ptr(hist), H, W, hist.size))

    def _run_query(self, plan, b, syms, prec):
        r = plan.roles
        col, thr, out, cnt = b[r["col"]], b[r["thr"]], b[r["out_vals"]], b[r["count"]]
        if out.size < col.size:
            raise ExecutionError(f"drain of {col.size} elements may overflow '{r['out_vals']}'")
        _lib.check(self._lib.sdfgb_host_query(_ptr(col), _ptr(thr), _ptr(out), _ptr(cnt), col.size,
                                              _lib.CMP[plan.params["op"]] | self._order_flag(), prec))

    def _order_flag(self):
        return _lib.QUERY_ORDERED if self.code.stream_order == "fifo" else 0

    def _run_spmv(self, plan, b, syms, prec):
        r = plan.roles
        rp, ci, v, x, y = (b[r[k]] for k in ("rowptr", "col", "val", "x", "b"))
        H = y.size
        nnz = ci.size
        if rp.size != H + 1:
            raise ExecutionError("row pointer length must be H + 1")
        if H and (rp[0] < 0 or rp[-1] > nnz or np.any(np.diff(rp) < 0)):
            raise ExecutionError("row pointers out of bounds for the column/value containers")
        if nnz and (ci.min() < 0 or ci.max() >= x.size):
            from .errors import OutOfBoundsError
            raise OutOfBoundsError(f"column index out of bounds for '{r['x']}' (size {x.size})")
        _lib.check(self._lib.sdfgb_host_spmv(_ptr(rp), _ptr(ci), _ptr(v), _ptr(x), _ptr(y), H, x.size,
                                             nnz, prec))

    def _run_jacobi2d(self, plan, b, syms, prec):
        A = b[plan.roles["A"]]
        N = int(X.evaluate(plan.params["N"], syms))
        T = int(X.evaluate(plan.params["steps"], syms))
        terms = plan.params["terms"]
        di = np.array([t[0] for t in terms], np.int32)
        dj = np.array([t[1] for t in terms], np.int32)
        _lib.check(self._lib.sdfgb_host_jacobi2d(_ptr(A), N, max(T, 0), plan.params["coef"], _ptr(di),
                                                 _ptr(dj), len(terms), prec))

    def _run_matmul(self, plan, b, syms, prec):
        A, B, C = b[plan.roles["A"]], b[plan.roles["B"]], b[plan.roles["C"]]
        M, K = plan.shape(plan.roles["A"], syms)
        N = plan.shape(plan.roles["B"], syms)[1]
        fn = self._lib.sdfgb_host_matmul_f64 if prec == _lib.PREC_NATIVE else self._lib.sdfgb_host_matmul
        _lib.check(fn(_ptr(A), _ptr(B), _ptr(C), M, N, K))


def compile_b200(sdfg: Any, precision: str = "fp32") -> CompiledB200Sdfg:
    """Convenience: classify + bind without a prior transformation pass."""
    code = generate(sdfg, require_marked=False)
    if code.precision != precision:
        code.precision = precision
    return invoke_toolchain(code)
