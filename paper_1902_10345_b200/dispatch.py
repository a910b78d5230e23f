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
import os
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
    prec = parts[1] if len(parts) > 1 else "native"
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


# ------------------------------------------------------- per-graph C shim

def _c_expr(e: X.Expr) -> str:
    """A symbol expression (container extents, loop counts) as C over the
    entry's int64_t symbol parameters (symbolic.py semantics: floor // and %)."""
    if isinstance(e, X.Num):
        if isinstance(e.value, float) and not float(e.value).is_integer():
            raise CodegenError(f"non-integer extent {e.value!r}")
        return f"((int64_t){int(e.value)})"
    if isinstance(e, X.Sym):
        return e.name
    if isinstance(e, X.Neg):
        return f"(-{_c_expr(e.arg)})"
    if isinstance(e, X.Bin) and e.op in ("+", "-", "*", "//", "%"):
        a, b = _c_expr(e.left), _c_expr(e.right)
        if e.op == "//":
            return f"sdfg_fdiv({a}, {b})"
        if e.op == "%":
            return f"sdfg_fmod({a}, {b})"
        return f"({a} {e.op} {b})"
    if isinstance(e, X.Call) and e.fn in ("min", "max") and e.args:
        out = _c_expr(e.args[0])
        for a in e.args[1:]:
            out = f"sdfg_{e.fn}({out}, {_c_expr(a)})"
        return out
    raise CodegenError(f"extent expression {e!r} has no C form")


def _c_num(v: float) -> str:
    return repr(float(v)) if float(v) == float(v) else "NAN"


def _size(plan: Plan, container: str, lo: int = 0, hi: Optional[int] = None) -> str:
    dims = plan.dims[container][lo:hi]
    return " * ".join(_c_expr(d) for d in dims) if dims else "((int64_t)1)"


def shim_source(plan: Plan, precision: str, order: str = "any") -> str:
    """The per-graph C translation unit: ``void <sdfg.name>(...)`` with the
    reference's exact signature -- non-transient containers in declaration
    order as ``double*`` / ``int64_t*``, then the symbols as ``int64_t``
    (codegen.py:620-627, :839-846) -- whose body calls the motif's host
    entry with the classified parameters baked in.  Like the reference's
    generated function it returns nothing; the entry's status is left for
    ``sdfgb_last_status()``."""
    r, pr = plan.roles, plan.params
    prec = "SDFGB_PREC_FP32" if precision == "fp32" else "SDFGB_PREC_NATIVE"
    m = plan.motif
    pre = ""
    if m == "histogram":
        call = (f"sdfgb_host_histogram({r['img']}, {r['hist']}, {_size(plan, r['img'], 0, 1)}, "
                f"{_size(plan, r['img'], 1)}, {_size(plan, r['hist'])}, {_c_num(pr['scale'])}, "
                f"{_c_num(pr['div'])}, {prec})")
    elif m == "histogram_int":
        call = (f"sdfgb_host_histogram_i64({r['img']}, {r['hist']}, {_size(plan, r['img'], 0, 1)}, "
                f"{_size(plan, r['img'], 1)}, {_size(plan, r['hist'])})")
    elif m == "query":
        flag = " | SDFGB_QUERY_ORDERED" if order == "fifo" else ""
        call = (f"sdfgb_host_query({r['col']}, {r['thr']}, {r['out_vals']}, {r['count']}, "
                f"{_size(plan, r['col'])}, {_CMP_C[pr['op']]}{flag}, {prec})")
    elif m == "spmv":
        call = (f"sdfgb_host_spmv({r['rowptr']}, {r['col']}, {r['val']}, {r['x']}, {r['b']}, "
                f"{_size(plan, r['b'])}, {_size(plan, r['x'])}, {_size(plan, r['col'])}, {prec})")
    elif m == "jacobi2d":
        terms = pr["terms"]
        pre = (f"    static const int32_t di[{len(terms)}] = {{{', '.join(str(t[0]) for t in terms)}}};\n"
               f"    static const int32_t dj[{len(terms)}] = {{{', '.join(str(t[1]) for t in terms)}}};\n"
               f"    const int64_t steps = {_c_expr(pr['steps'])};\n")
        call = (f"sdfgb_host_jacobi2d({r['A']}, {_c_expr(pr['N'])}, steps > 0 ? steps : 0, "
                f"{_c_num(pr['coef'])}, di, dj, {len(terms)}, {prec})")
    elif m == "matmul":
        fn = "sdfgb_host_matmul" if precision == "fp32" else "sdfgb_host_matmul_f64"
        call = (f"{fn}({r['A']}, {r['B']}, {r['C']}, {_size(plan, r['A'], 0, 1)}, "
                f"{_size(plan, r['B'], 1, 2)}, {_size(plan, r['A'], 1, 2)})")
    else:
        raise CodegenError(f"no host entry for motif '{m}'")
    params = [f"{_CT[t]}* {n}" for n, t in plan.pointer_args] + [f"int64_t {sym}" for sym in plan.symbol_args]
    unused = "".join(f"    (void){sym};\n" for sym in plan.symbol_args)
    return (_describe(plan, precision)
            + "#include <math.h>\n#include <stdint.h>\n#include \"sdfgb200.h\"\n\n"
            + "static inline int64_t sdfg_fdiv(int64_t a, int64_t b) { int64_t q = a / b; "
              "return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q; }\n"
            + "static inline int64_t sdfg_fmod(int64_t a, int64_t b) { int64_t r = a % b; "
              "return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r; }\n"
            + "static inline int64_t sdfg_min(int64_t a, int64_t b) { return a < b ? a : b; }\n"
            + "static inline int64_t sdfg_max(int64_t a, int64_t b) { return a > b ? a : b; }\n\n"
            + f"void {plan.name}({', '.join(params)}) {{\n{unused}{pre}    {call};\n}}\n")


_CMP_C = {"<": "SDFGB_CMP_LT", "<=": "SDFGB_CMP_LE", ">": "SDFGB_CMP_GT", ">=": "SDFGB_CMP_GE",
          "==": "SDFGB_CMP_EQ", "!=": "SDFGB_CMP_NE"}


def shim_link_flags() -> list:
    """Extra flags with which the reference's own ``invoke_toolchain(code,
    flags)`` (codegen.py:890-913; it inserts them after ``cc``) compiles a
    B200 shim: the header, and libsdfgb200.so as a forced dependency."""
    libdir = os.path.dirname(_lib.LIB_PATH)
    return ["-I", os.path.dirname(_lib.HEADER), "-Wl,--no-as-needed", "-L", libdir, "-l:libsdfgb200.so",
            f"-Wl,-rpath,{libdir}"]


def build_shim(code: "GeneratedB200Code") -> str:
    """cc -shared -fPIC -O2 (the reference's toolchain, codegen.py:890-913)
    of the shim, linked against libsdfgb200.so; cached in _gen/ by digest."""
    import hashlib
    import shutil
    import subprocess
    import threading
    from .generic import GEN_DIR
    cc = os.environ.get("CC") or shutil.which("cc") or shutil.which("gcc")
    if not cc:
        raise ToolchainError("no C compiler (cc) for the drop-in shim")
    if not os.path.exists(_lib.LIB_PATH):
        raise ToolchainError(f"{_lib.LIB_PATH} is not built; run __graft_entry__.build()")
    inc = os.path.dirname(_lib.HEADER)
    libdir = os.path.dirname(_lib.LIB_PATH)
    flags = ["-shared", "-fPIC", "-O2", "-I", inc]
    key = hashlib.sha256((code.source + " ".join(flags)).encode()).hexdigest()[:16]
    os.makedirs(GEN_DIR, exist_ok=True)
    base = os.path.join(GEN_DIR, f"shim_{code.name}_{key}")
    so = base + ".so"
    if os.path.exists(so):
        return so
    tag = f"{os.getpid()}.{threading.get_ident()}"
    src, tmp = f"{base}.{tag}.c", f"{so}.{tag}.tmp"
    with open(src, "w") as f:
        f.write(code.source)
    # $ORIGIN/..: the shim finds the library next to the package wherever the
    # tree was copied (the GPU boxes run a copy)
    cmd = [cc] + flags + ["-o", tmp, src, "-L", libdir, "-l:libsdfgb200.so", "-Wl,-rpath,$ORIGIN/.."]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise ToolchainError(f"cc failed for the '{code.name}' shim:\n{r.stderr}")
    os.replace(src, base + ".c")
    os.replace(tmp, so)
    return so


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
        mode = ("native", "any")
    prec, order = mode
    if prec not in PRECISIONS:
        raise CodegenError(f"unknown precision '{prec}'")
    if order not in STREAM_ORDERS:
        raise CodegenError(f"unknown stream order '{order}'")
    return GeneratedB200Code(shim_source(plan, prec, order), g.name, plan.pointer_args, plan.symbol_args,
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
    """Build and load the graph's shim (the reference compiles its generated
    C with cc here, codegen.py:890-913); the kernels themselves are the
    prebuilt sm_100a library.  Generic programs are compiled with nvcc for
    sm_100a (generic.py)."""
    if code.lowered is not None:
        from .generic import GenericProgram, build
        return GenericProgram(code.graph, code.lowered, build(code.lowered))
    try:
        lib = _lib.load()
    except _lib.BackendUnavailable as exc:
        raise ToolchainError(str(exc)) from exc
    return CompiledB200Sdfg(code, lib, build_shim(code))


class CompiledB200Sdfg:
    """A loaded B200 program; ``run`` has CompiledSdfg.run's contract and
    makes the reference's own call: ``getattr(lib, code.name)(*ptrs, *syms)``
    (codegen.py:866-887), then reads the entry's status."""

    def __init__(self, code: GeneratedB200Code, lib, shim_path: str):
        self.code = code
        self._lib = lib
        self.shim_path = shim_path
        self._shim = ctypes.CDLL(shim_path)
        self._fn = getattr(self._shim, code.name)
        self._fn.restype = None
        self._fn.argtypes = [ctypes.c_void_p] * len(code.pointer_args) + [ctypes.c_int64] * len(code.symbol_args)

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
        r = plan.roles
        if plan.motif == "query" and bufs[r["out_vals"]].size < bufs[r["col"]].size:
            raise ExecutionError(f"drain of {bufs[r['col']].size} elements may overflow '{r['out_vals']}'")
        if plan.motif == "spmv" and bufs[r["rowptr"]].size != bufs[r["b"]].size + 1:
            raise ExecutionError("row pointer length must be H + 1")
        self._fn(*[b.ctypes.data for b in bufs.values()], *[syms[s] for s in plan.symbol_args])
        _lib.check(self._lib.sdfgb_last_status())
        return bufs


def compile_b200(sdfg: Any, precision: str = "native") -> CompiledB200Sdfg:
    """Convenience: classify + bind without a prior transformation pass."""
    code = generate(sdfg, require_marked=False)
    if code.plan is not None and code.precision != precision:
        code.precision = precision
        code.source = shim_source(code.plan, precision, code.stream_order)
    return invoke_toolchain(code)
