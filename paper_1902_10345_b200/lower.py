"""Generic Map/tasklet -> CUDA lowering.

The five motif kernels cover the BASELINE workloads; every other SDFG the
reference can express with maps, tasklets, WCR memlets, stream pushes,
indirection, nested graphs and interstate control flow is lowered here to
one CUDA translation unit for sm_100a, compiled with nvcc and called
through the same C-ABI shape as the reference's generated C
(codegen.py:615-660): one ``extern "C"`` entry taking the non-transient
containers in declaration order and the symbols.

Semantics follow the reference's CPU dispatcher and interpreter, re-stated
for a GPU (not translated from them):

* a top-level Map scope becomes one kernel: a grid-stride loop over the
  flattened map range (ranges are inclusive, ``begin:end:stride``,
  symbolic.py:579-618); nested maps become loops inside the thread
  (codegen.py:500-524 emits the same nest sequentially);
* Map iterations are concurrent, so WCR writes from inside a map are device
  atomics (sum/product/min/max, ir.py:89-121); plain writes keep the
  program's own race semantics, as the reference's ``cpu_parallel``
  schedule does;
* a transient whose every access lies inside one top-level map is private
  to the map iteration (registers/local memory, zero-initialised like the
  reference's ``calloc``, codegen.py:637-641); other transients live in HBM;
* a stream push reserves a slot with one atomic on the stream's counter
  (order unspecified: a Stream is a concurrent queue); a
  drain copies the queue's contents to the start of the target array
  (interpreter.py:279-287);
* tasklet bodies are translated from their Python subset (tasklets.py:1-12)
  with the reference's typing rules: int64/float64 connectors, ``/`` is
  real division, ``//`` and ``%`` floor (sdfg_fdiv/sdfg_fmod), float ``//``
  is floor of the real quotient, assigning a float to an int64 output
  truncates (tasklets.py:348-514);
* subscript writes index the whole flattened container and are bounds-
  checked (interpreter.py:262-268 raises OutOfBoundsError); subscript reads
  index the memlet's block from its origin;
* a nested SDFG inside a map is a __device__ function running its own state
  machine per map iteration (codegen.py:573-595 emits a static C function);
* the top-level state machine runs on the host: conditions over symbols are
  host arithmetic, conditions over size-1 containers read them back.

* a consume scope draining its stream (``size(S) > 0``) is a persistent
  work-queue kernel: tickets, per-item ready flags, and quiescence when every
  pushed item has finished (codegen.py:526-543 runs P sequential workers).

* a vectorised memlet (tile > 1 on the last dimension, Vectorization) runs
  the tasklet once per lane.

* a custom WCR (ir.py:100-121) becomes a __device__ combine function
  translated from its tasklet, applied with a compare-and-swap loop.

Not lowered (CodegenError): other consume conditions, symbolic vector
widths, stream pops outside consume scopes.
"""

from __future__ import annotations

import ast
import hashlib
from dataclasses import dataclass, field
from typing import Optional

from . import expr as X
from .errors import CodegenError
from .graph import Graph, State, from_json

CT = {"int64": "int64_t", "float64": "double"}
MAX_PRIVATE = 4096  # elements of a per-iteration private transient
QUEUE_ITEMS = int(__import__("os").environ.get("SDFGB_GEN_QUEUE", 1 << 22))  # work-queue stream capacity


class LoweringError(CodegenError):
    pass


def _ident(s: str) -> str:
    return "".join(c if c.isalnum() else "_" for c in s)


# ------------------------------------------------------------------ helpers

PRELUDE = r"""
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

#define GEN_DEV __device__ __forceinline__
#define GEN_HD __host__ __device__ __forceinline__

GEN_HD int64_t g_fdiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
GEN_HD int64_t g_fmod(int64_t a, int64_t b) {
    int64_t r = a % b;
    return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r;
}
GEN_HD int64_t g_imin(int64_t a, int64_t b) { return a < b ? a : b; }
GEN_HD int64_t g_imax(int64_t a, int64_t b) { return a > b ? a : b; }
GEN_HD int64_t g_iabs(int64_t a) { return a < 0 ? -a : a; }
// number of points of the inclusive range begin:end:stride
GEN_HD int64_t g_rlen(int64_t b, int64_t e, int64_t s) {
    if (s > 0) return e < b ? 0 : (e - b) / s + 1;
    if (s < 0) return e > b ? 0 : (b - e) / (-s) + 1;
    return 0;
}

// write-conflict resolution on memory other threads may touch
GEN_DEV void wcr_sum(double* p, double v) { atomicAdd(p, v); }
GEN_DEV void wcr_sum(int64_t* p, int64_t v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}
template <typename T, typename F>
GEN_DEV void wcr_cas(T* p, T v, F f) {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(p);
    unsigned long long old = *a, assumed;
    do {
        assumed = old;
        T cur;
        memcpy(&cur, &assumed, 8);
        T nv = f(cur, v);
        unsigned long long nb;
        memcpy(&nb, &nv, 8);
        old = atomicCAS(a, assumed, nb);
    } while (old != assumed);
}
GEN_DEV void wcr_product(double* p, double v) { wcr_cas(p, v, [](double a, double b) { return a * b; }); }
GEN_DEV void wcr_product(int64_t* p, int64_t v) { wcr_cas(p, v, [](int64_t a, int64_t b) { return a * b; }); }
GEN_DEV void wcr_min(double* p, double v) { wcr_cas(p, v, [](double a, double b) { return b < a ? b : a; }); }
GEN_DEV void wcr_max(double* p, double v) { wcr_cas(p, v, [](double a, double b) { return b > a ? b : a; }); }
GEN_DEV void wcr_min(int64_t* p, int64_t v) { atomicMin(reinterpret_cast<long long*>(p), (long long)v); }
GEN_DEV void wcr_max(int64_t* p, int64_t v) { atomicMax(reinterpret_cast<long long*>(p), (long long)v); }
// the same resolutions on thread-private memory
template <typename T> GEN_HD void pwcr_sum(T* p, T v) { *p = *p + v; }
template <typename T> GEN_HD void pwcr_product(T* p, T v) { *p = *p * v; }
template <typename T> GEN_HD void pwcr_min(T* p, T v) { *p = v < *p ? v : *p; }
template <typename T> GEN_HD void pwcr_max(T* p, T v) { *p = v > *p ? v : *p; }

// first error wins: 1 = out-of-bounds subscript write, 2 = out-of-bounds
// subscript read, 3 = stream overflow, 4 = drain overflows its target,
// 5 = a consume worker waited past its watchdog, 6 = a memlet index outside
// its container (OutOfBoundsError, interpreter.py:216-233)
GEN_DEV void gen_fail(int* err, int code) { atomicCAS(err, 0, code); }

template <typename T>
GEN_DEV void stream_push(T* buf, unsigned long long* cnt, int64_t cap, T v, int* err) {
    const unsigned long long i = atomicAdd(cnt, 1ull);
    if ((int64_t)i < cap) buf[i] = v; else gen_fail(err, 3);
}

// work-queue streams (consumed by a consume scope): items carry a ready
// flag; q[0] = next ticket, q[1] = items finished (pushes of an item happen
// before it counts as finished, so finished == pushed means quiescence)
GEN_DEV unsigned ld_acq_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
GEN_DEV unsigned long long ld_acq_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <typename T>
GEN_DEV void stream_push_q(T* buf, unsigned long long* cnt, int64_t cap, unsigned* ready,
                           unsigned long long* q, T v, int* err) {
    const unsigned long long i = atomicAdd(cnt, 1ull);
    if ((int64_t)i < cap) {
        buf[i] = v;
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + i), "r"(1u) : "memory");
    } else {
        gen_fail(err, 3);
        atomicAdd(q + 1, 1ull);  // the lost item counts as finished: quiescence stays reachable
    }
}
__global__ void gen_queue_reset(unsigned* ready, unsigned long long* cnt, unsigned long long* q, int64_t cap) {
    const unsigned long long n = *cnt;
    const int64_t m = (int64_t)n < cap ? (int64_t)n : cap;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        ready[i] = 0u;
}

template <typename T>
__global__ void gen_drain(const T* __restrict__ buf, const unsigned long long* __restrict__ cnt, T* dst,
                          int64_t dst_size, int* err) {
    const int64_t n = (int64_t)*cnt;
    if (n > dst_size) {
        if (blockIdx.x == 0 && threadIdx.x == 0) gen_fail(err, 4);
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = buf[i];
}

// ExecutionReport builds: add a device-resident count (a stream's items) to a slot
__global__ void gen_rep_addp(unsigned long long* slot, const unsigned long long* v) { *slot += *v; }

static int gen_blocks(int64_t total) {
    int64_t b = (total + 255) / 256;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}
// A map kernel launched with programmatic dependent launch: its CTAs are
// scheduled while the previous kernel of the stream drains; every generated
// kernel starts with griddepcontrol.wait, so nothing is read or written
// before that kernel has completed.
template <typename... P, typename... A>
static cudaError_t gen_launch(void (*k)(P...), int grid, int block, cudaStream_t st, A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.stream = st;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}
// Keep stream-ordered allocations cached between runs: with the default
// release threshold (0) every synchronize hands the pool back to the driver
// and the next cudaMallocAsync pays a real allocation (ms-scale, variable).
static void gen_pool_keep() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done = true;
}
// Per-thread, per-device error word and pinned status word, kept across
// runs: a run costs one memset and one 4-byte copy instead of an
// allocation, a pageable copy and two synchronisations (reentrant: one
// run per thread at a time, like the reference's C entry)
static int* gen_err_dev() {
    static thread_local int* cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (!cache[dev] && cudaMalloc((void**)&cache[dev], 16) != cudaSuccess) cache[dev] = nullptr;
    return cache[dev];
}
static int* gen_status_host() {
    static thread_local int* h = nullptr;
    if (!h && cudaHostAlloc((void**)&h, 16, cudaHostAllocDefault) != cudaSuccess) h = nullptr;
    return h;
}
template <typename T>
static T gen_read(const T* p, cudaStream_t s) {
    T v;
    cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return v;
}
"""


# ------------------------------------------------------------------ expressions

class Env:
    """Name resolution for symbolic expressions: map parameters, symbols,
    size-1 containers (their element 0) and stream sizes."""

    def __init__(self, lw: "Lowering", params: dict, host: bool):
        self.lw = lw
        self.params = params  # map param -> C name
        self.host = host

    def child(self, more: dict) -> "Env":
        p = dict(self.params)
        p.update(more)
        return Env(self.lw, p, self.host)

    def sym(self, name: str) -> str:
        if name in self.params:
            return self.params[name]
        if name in self.lw.sym_names:
            return f"s_{_ident(name)}"
        d = self.lw.g.data.get(name)
        if d is not None and d.kind == "array" and self.lw.static_size(d) == 1:
            if self.host:
                return f"gen_read({self.lw.cname(name)}, st)"
            return f"{self.lw.cname(name)}[0]"
        raise LoweringError(f"unbound name '{name}' in an expression of '{self.lw.g.name}'")

    def emit(self, e: X.Expr) -> str:
        if isinstance(e, X.Num):
            v = e.value
            if isinstance(v, float):
                return repr(v)
            return f"{int(v)}LL"
        if isinstance(e, X.Sym):
            return self.sym(e.name)
        if isinstance(e, X.Neg):
            return f"(-{self.emit(e.arg)})"
        if isinstance(e, X.Bin):
            a, b = self.emit(e.left), self.emit(e.right)
            if e.op == "//":
                return f"g_fdiv({a}, {b})"
            if e.op == "%":
                return f"g_fmod({a}, {b})"
            if e.op == "/":
                return f"((double)({a}) / (double)({b}))"
            return f"({a} {e.op} {b})"
        if isinstance(e, X.Call):
            if e.fn == "size":
                s = e.args[0].name
                if self.host:
                    return f"(int64_t)gen_read(n_{_ident(s)}, st)"
                return f"(int64_t)(*n_{_ident(s)})"
            fn = "g_imin" if e.fn == "min" else "g_imax"
            out = self.emit(e.args[0])
            for a in e.args[1:]:
                out = f"{fn}({out}, {self.emit(a)})"
            return out
        if isinstance(e, X.Cmp):
            return f"({self.emit(e.left)} {e.op} {self.emit(e.right)})"
        if isinstance(e, X.BoolOp):
            op = " && " if e.op == "and" else " || "
            return "(" + op.join(self.emit(a) for a in e.args) + ")"
        if isinstance(e, X.Not):
            return f"(!{self.emit(e.arg)})"
        raise LoweringError(f"cannot lower expression {e!r}")


# ------------------------------------------------------------------ tasklets

_BIN = {ast.Add: "+", ast.Sub: "-", ast.Mult: "*", ast.Div: "/", ast.FloorDiv: "//", ast.Mod: "%"}
_CMP = {ast.Lt: "<", ast.LtE: "<=", ast.Gt: ">", ast.GtE: ">=", ast.Eq: "==", ast.NotEq: "!="}


class TaskletC:
    """Python-subset tasklet body -> C statements (types as tasklets.py:352-400)."""

    def __init__(self, body: list, types: dict, names: dict, array_reads: dict, array_writes: dict,
                 outputs: set, dynamic: set):
        self.body = body
        self.types = types            # connector -> basetype
        self.names = names            # connector -> C variable
        self.array_reads = array_reads    # connector -> (pointer, size expr)
        self.array_writes = array_writes  # connector -> (pointer, size expr, wcr, private)
        self.outputs = outputs
        self.dynamic = dynamic        # outputs needing a __set flag
        self.locals: dict[str, str] = {}
        self.wcount: dict[str, str] = {}  # connector -> C counter of its subscript writes (report builds)
        self._infer(body)

    def type_of(self, n: ast.expr) -> str:
        if isinstance(n, ast.Constant):
            return "float64" if isinstance(n.value, float) else "int64"
        if isinstance(n, ast.Name):
            if n.id in self.types:
                return self.types[n.id]
            if n.id in self.locals:
                return self.locals[n.id]
            raise LoweringError(f"tasklet: unknown name '{n.id}'")
        if isinstance(n, ast.BinOp):
            if isinstance(n.op, ast.Div):
                return "float64"
            return "float64" if "float64" in (self.type_of(n.left), self.type_of(n.right)) else "int64"
        if isinstance(n, ast.UnaryOp):
            return "int64" if isinstance(n.op, ast.Not) else self.type_of(n.operand)
        if isinstance(n, (ast.BoolOp, ast.Compare)):
            return "int64"
        if isinstance(n, ast.IfExp):
            return "float64" if "float64" in (self.type_of(n.body), self.type_of(n.orelse)) else "int64"
        if isinstance(n, ast.Subscript):
            return self.type_of(n.value)
        if isinstance(n, ast.Call):
            if n.func.id == "abs":
                return self.type_of(n.args[0])
            return "float64" if any(self.type_of(a) == "float64" for a in n.args) else "int64"
        raise LoweringError(f"tasklet: cannot type {type(n).__name__}")

    def _infer(self, stmts: list) -> None:
        for s in stmts:
            if isinstance(s, ast.Assign) and isinstance(s.targets[0], ast.Name):
                name = s.targets[0].id
                if name in self.types:
                    continue
                t = self.type_of(s.value)
                prev = self.locals.get(name)
                self.locals[name] = "float64" if "float64" in (prev, t) else t
            elif isinstance(s, ast.If):
                self._infer(s.body)
                self._infer(s.orelse)

    def var(self, name: str) -> str:
        if name in self.names:
            return self.names[name]
        if name in self.locals:
            return f"l_{_ident(name)}"
        raise LoweringError(f"tasklet: unknown name '{name}'")

    def ex(self, n: ast.expr) -> str:
        if isinstance(n, ast.Constant):
            if isinstance(n.value, bool):
                return "1LL" if n.value else "0LL"
            if isinstance(n.value, float):
                return repr(n.value)
            return f"{n.value}LL"
        if isinstance(n, ast.Name):
            return self.var(n.id)
        if isinstance(n, ast.BinOp):
            op = _BIN[type(n.op)]
            a, b = self.ex(n.left), self.ex(n.right)
            fl = "float64" in (self.type_of(n.left), self.type_of(n.right))
            if op == "/":
                return f"((double)({a}) / (double)({b}))"
            if op == "//":
                return f"floor((double)({a}) / (double)({b}))" if fl else f"g_fdiv({a}, {b})"
            if op == "%":
                if fl:
                    raise LoweringError("float modulo is not supported in generated code")
                return f"g_fmod({a}, {b})"
            return f"({a} {op} {b})"
        if isinstance(n, ast.UnaryOp):
            if isinstance(n.op, ast.USub):
                return f"(-{self.ex(n.operand)})"
            if isinstance(n.op, ast.UAdd):
                return self.ex(n.operand)
            return f"((int64_t)!({self.ex(n.operand)}))"
        if isinstance(n, ast.BoolOp):
            op = " && " if isinstance(n.op, ast.And) else " || "
            return "((int64_t)(" + op.join(f"({self.ex(v)})" for v in n.values) + "))"
        if isinstance(n, ast.Compare):
            return f"((int64_t)({self.ex(n.left)} {_CMP[type(n.ops[0])]} {self.ex(n.comparators[0])}))"
        if isinstance(n, ast.IfExp):
            t = CT[self.type_of(n)]
            return f"(({self.ex(n.test)}) ? ({t})({self.ex(n.body)}) : ({t})({self.ex(n.orelse)}))"
        if isinstance(n, ast.Subscript):
            name = n.value.id
            if name not in self.array_reads:
                raise LoweringError(f"tasklet: subscript read of '{name}' without an array memlet")
            ptr, size = self.array_reads[name]
            return f"g_rd({ptr}, (int64_t)({self.ex(n.slice)}), {size}, g_err)"
        if isinstance(n, ast.Call):
            args = [self.ex(a) for a in n.args]
            if n.func.id == "abs":
                return f"fabs({args[0]})" if self.type_of(n.args[0]) == "float64" else f"g_iabs({args[0]})"
            fl = any(self.type_of(a) == "float64" for a in n.args)
            fn = ("fmin" if n.func.id == "min" else "fmax") if fl else ("g_imin" if n.func.id == "min" else "g_imax")
            out = f"(double)({args[0]})" if fl else args[0]
            for a in args[1:]:
                out = f"{fn}({out}, {'(double)(' + a + ')' if fl else a})"
            return out
        raise LoweringError(f"tasklet: cannot lower {type(n).__name__}")

    def stmt(self, s, ind: str, out: list) -> None:
        if isinstance(s, ast.Assign):
            tgt = s.targets[0]
            val = self.ex(s.value)
            if isinstance(tgt, ast.Name):
                name = tgt.id
                tt = self.types.get(name) or self.locals.get(name)
                if tt == "int64" and self.type_of(s.value) == "float64":
                    val = f"(int64_t)({val})"
                out.append(f"{ind}{self.var(name)} = {val};")
                if name in self.dynamic:
                    out.append(f"{ind}{self.var(name)}__set = 1;")
            else:
                name = tgt.value.id
                ptr, size, wcr, private = self.array_writes[name]
                idx = self.ex(tgt.slice)
                fn = "g_wr" if wcr is None else f"g_wr_{'p' if private else ''}{wcr}"
                out.append(f"{ind}{fn}({ptr}, (int64_t)({idx}), {size}, ({CT[self.types[name]]})({val}), g_err);")
                if name in self.wcount:
                    out.append(f"{ind}++{self.wcount[name]};")
            return
        if isinstance(s, ast.If):
            out.append(f"{ind}if ({self.ex(s.test)}) {{")
            for b in s.body:
                self.stmt(b, ind + "    ", out)
            if s.orelse:
                out.append(f"{ind}}} else {{")
                for b in s.orelse:
                    self.stmt(b, ind + "    ", out)
            out.append(f"{ind}}}")
            return
        raise LoweringError(f"tasklet: unsupported statement {type(s).__name__}")

    def emit(self, ind: str) -> list:
        out = [f"{ind}{CT[t]} l_{_ident(n)} = 0;" for n, t in sorted(self.locals.items())]
        for s in self.body:
            self.stmt(s, ind, out)
        return out


SUBSCRIPT_HELPERS = r"""
template <typename T>
GEN_DEV T g_rd(const T* p, int64_t i, int64_t n, int* err) {
    if (i < 0 || i >= n) { gen_fail(err, 2); return T(0); }
    return p[i];
}
template <typename T>
GEN_DEV void g_wr(T* p, int64_t i, int64_t n, T v, int* err) {
    if (i < 0 || i >= n) { gen_fail(err, 1); return; }
    p[i] = v;
}
#define GEN_WR(kind, fn)                                                        \
    template <typename T>                                                       \
    GEN_DEV void g_wr_##kind(T* p, int64_t i, int64_t n, T v, int* err) {       \
        if (i < 0 || i >= n) { gen_fail(err, 1); return; }                      \
        fn(p + i, v);                                                           \
    }
GEN_WR(sum, wcr_sum)
GEN_WR(product, wcr_product)
GEN_WR(min, wcr_min)
GEN_WR(max, wcr_max)
GEN_WR(psum, pwcr_sum)
GEN_WR(pproduct, pwcr_product)
GEN_WR(pmin, pwcr_min)
GEN_WR(pmax, pwcr_max)
"""


# ------------------------------------------------------------------ lowering

@dataclass
class Lowered:
    name: str
    source: str
    entry: str
    pointer_args: list
    symbol_args: list
    digest: str = ""
    notes: list = field(default_factory=list)
    # ExecutionReport builds (lower(g, report=True)): counter slot -> key
    # ("<state>:e<id>", nested "<graph>/<state>:e<id>", "__tasklets"), and
    # the state index order of the visit log
    report_keys: Optional[list] = None
    state_names: Optional[list] = None


class Lowering:
    def __init__(self, g: Graph, fn_prefix: str = "gen", nested: bool = False, report: Optional[dict] = None,
                 keyprefix: str = ""):
        self.g = g
        self.prefix = fn_prefix
        self.nested = nested
        # ExecutionReport build: {"slots": {key: index}} shared with nested
        # lowerings; None for the normal (timed) build, which has no counters
        self.rep = report
        self.keyprefix = keyprefix
        assigned = {a for t in g.transitions for a, _ in t.assignments}
        self.sym_names = list(g.symbols) + sorted(assigned - set(g.symbols))
        self.kernels: list[str] = []
        self.devfns: list[str] = []
        self.kcount = 0
        self.tcount = 0
        # bounds-check hoisting (top_map): accesses recorded while a map body
        # is emitted, and the mode that emits it without per-access checks
        self.track = None
        self.unchecked = False
        self.scoped: dict = {}  # transient -> (state, top entry): thread-sliced per-iteration scratch
        self.private = self._find_private()
        self.consumed = set()
        for st in g.states:
            for n in st.nodes:
                if n.kind == "consume_entry":
                    for e in st.in_edges(n.id):
                        if e.dst_conn == "IN_stream" and not e.memlet.is_empty:
                            self.consumed.add(e.memlet.data)
        self.pop_vars: dict = {}  # stream -> C variable of the element a consume worker popped
        self.custom_wcr: dict = {}

    # -- containers ---------------------------------------------------------

    def cname(self, data: str) -> str:
        return f"c_{_ident(data)}"

    def static_size(self, d) -> Optional[int]:
        total = 1
        for dim in d.dims:
            try:
                total *= int(X.evaluate(dim, {}))
            except X.ExprError:
                return None
        return total

    def flat(self, data: str, idx: list, env: Env) -> str:
        d = self.g.data[data]
        if len(idx) != len(d.dims):
            raise LoweringError(f"rank mismatch on '{data}'")
        out = idx[0]
        for k in range(1, len(d.dims)):
            out = f"(({out}) * ({env.emit(d.dims[k])}) + ({idx[k]}))"
        return out

    def in_bounds(self, data: str, idx: list, env: Env) -> str:
        """Every index inside its dimension (the interpreter checks each
        access, interpreter.py:216-233; the C path does not)."""
        d = self.g.data[data]
        return " && ".join(f"(uint64_t)({i}) < (uint64_t)({env.emit(dim)})" for i, dim in zip(idx, d.dims))

    def _track(self, data: str, subset, width: int) -> None:
        if self.track is not None:
            self.track.append((data, [r.begin for r in subset]) if width == 1 else None)

    def size_expr(self, data: str, env: Env) -> str:
        d = self.g.data[data]
        return "(" + " * ".join(f"({env.emit(x)})" for x in d.dims) + ")"

    def origin(self, data: str, subset, env: Env) -> str:
        return self.flat(data, [env.emit(r.begin) for r in subset], env)

    def block_size(self, subset, env: Env) -> str:
        return "(" + " * ".join(f"g_rlen({env.emit(r.begin)}, {env.emit(r.end)}, 1)" for r in subset) + ")"

    def _find_private(self) -> set:
        """Transients whose every access node sits inside one top-level map
        (same state, same entry): per-iteration private storage."""
        owner: dict[str, set] = {}
        for st in self.g.states:
            parent = st.scope_parent()
            for n in st.nodes:
                if n.kind != "access":
                    continue
                top = parent[n.id]
                while top is not None and parent[top] is not None:
                    top = parent[top]
                owner.setdefault(n.data, set()).add((st.name, top))
        out = set()
        for name, owners in owner.items():
            d = self.g.data.get(name)
            if d is None or not d.transient or d.kind != "array":
                continue
            if len(owners) == 1 and next(iter(owners))[1] is not None:
                sz = self.static_size(d)
                if sz is not None and sz <= MAX_PRIVATE:
                    out.add(name)
                else:
                    # symbolic or large: each thread of the owning map's grid gets
                    # its own slice of one HBM buffer (iterations run concurrently;
                    # the reference's sequential loop shares one buffer)
                    self.scoped[name] = next(iter(owners))
        return out

    # -- parameters ----------------------------------------------------------

    def kparams(self) -> str:
        ps = []
        for name, d in self.g.data.items():
            if name in self.private:
                continue
            if d.kind == "stream":
                ps += [f"{CT[d.basetype]}* {self.cname(name)}", f"unsigned long long* n_{_ident(name)}",
                       f"int64_t cap_{_ident(name)}"]
                if name in self.consumed:
                    ps += [f"unsigned* r_{_ident(name)}", f"unsigned long long* q_{_ident(name)}"]
            else:
                ps.append(f"{CT[d.basetype]}* {self.cname(name)}")
        ps += [f"int64_t s_{_ident(s)}" for s in self.sym_names]
        ps.append("int* g_err")
        if self.rep is not None:
            ps.append("unsigned long long* g_rep")
        return ", ".join(ps)

    def kargs(self) -> str:
        a = []
        for name, d in self.g.data.items():
            if name in self.private:
                continue
            if d.kind == "stream":
                a += [self.cname(name), f"n_{_ident(name)}", f"cap_{_ident(name)}"]
                if name in self.consumed:
                    a += [f"r_{_ident(name)}", f"q_{_ident(name)}"]
            else:
                a.append(self.cname(name))
        a += [f"s_{_ident(s)}" for s in self.sym_names]
        a.append("g_err")
        if self.rep is not None:
            a.append("g_rep")
        return ", ".join(a)

    # -- ExecutionReport counters (interpreter.py:369-382, 514-545) -----------
    # Every memlet edge counts what the interpreter's _produce counts: the
    # memlet's `accesses` when it has one, else the actual elements -- the
    # block a scope instance or access node reads, one per scalar a tasklet
    # assigns (zero when a dynamic output stays unassigned), one per subscript
    # write, the items a stream drain moves -- and an exit edge sums what
    # crosses it.  Scope-level counts are atomics on the device; counts of
    # top-level nodes are host additions once per state visit.

    def slot(self, key: str) -> int:
        slots = self.rep["slots"]
        return slots.setdefault(key, len(slots))

    def ekey(self, st: State, e) -> str:
        return f"{self.keyprefix}{st.name}:e{e.id}"

    def dcount(self, key: str, expr: str, ind: str, out: list) -> None:
        if self.rep is None:
            return
        k = self.slot(key)
        if expr != "0":
            out.append(f"{ind}atomicAdd(&g_rep[{k}], (unsigned long long)({expr}));")

    def hcount(self, key: str, expr: str, out: list) -> None:
        if self.rep is None:
            return
        k = self.slot(key)
        if expr != "0":
            out.append(f"    g_reph[{k}] += (unsigned long long)({expr});")

    def vol(self, subset, env: Env) -> str:
        if not subset:
            return "1LL"
        return "(" + " * ".join(f"g_rlen({env.emit(r.begin)}, {env.emit(r.end)}, {env.emit(r.stride)}) * "
                                f"({env.emit(r.tile)})" for r in subset) + ")"

    def exit_chain(self, st: State, e) -> list:
        """Edges a value committed on ``e`` crosses after it: scope exits
        (the interpreter's _boundary_actual) and local-stream forwards."""
        dst = st.nodes[e.dst]
        out = []
        if dst.kind == "access":
            d = self.g.data.get(dst.data)
            if d is not None and d.kind == "stream" and d.transient:
                for o in st.out_edges(dst.id):
                    if st.nodes[o.dst].kind in ("map_exit", "consume_exit") and o.dst_conn:
                        out.append(o)
                        out += self.exit_chain(st, o)
            return out
        if dst.kind in ("map_exit", "consume_exit") and e.dst_conn:
            conn = "OUT_" + e.dst_conn[3:]
            for nxt in st.out_edges(dst.id):
                if nxt.src_conn == conn:
                    out.append(nxt)
                    out += self.exit_chain(st, nxt)
        return out

    def chain_counts(self, st: State, e, actual: str, ind: str, out: list) -> None:
        for c in self.exit_chain(st, e):
            if c.memlet.accesses is None and not c.memlet.is_empty:
                self.dcount(self.ekey(st, c), actual, ind, out)

    def instance_counts(self, st: State, n, env: Env, ind: str, out: list) -> None:
        """One scope instance: the block every entry edge reads (:514-536)."""
        if self.rep is None:
            return
        for e in st.out_edges(n.id):
            m = e.memlet
            if m.is_empty:
                v = "0"
            elif n.kind == "consume_entry" and e.src_conn == "OUT_stream":
                v = "1"
            elif self.g.data[m.data].kind == "stream":
                v = "0"
            else:
                v = self.vol(m.subset, env)
            self.dcount(self.ekey(st, e), v, ind, out)

    def access_counts(self, st: State, n, env: Env, ind: str, out: list, host: bool) -> None:
        """An access node firing (_fire_access / _fire_stream_access)."""
        if self.rep is None:
            return
        stream = self.g.data[n.data].kind == "stream"
        for e in st.out_edges(n.id):
            m = e.memlet
            key = self.ekey(st, e)
            dkind = st.nodes[e.dst].kind
            if m.is_empty:
                v = "0"
            elif m.accesses is not None:
                v = env.emit(m.accesses)
            elif stream:
                # drains count their items where they run (top_access / the
                # forwarded pushes); handles into a scope move nothing
                v = "0"
            else:
                v = self.vol(m.subset, env)
                if dkind in ("map_exit", "consume_exit") and not host:
                    self.chain_counts(st, e, v, ind, out)
            if host:
                self.hcount(key, v, out)
            else:
                self.dcount(key, v, ind, out)

    def exit_of(self, st: State, entry_id: int):
        for x in st.nodes:
            if x.kind in ("map_exit", "consume_exit") and x.doc.get("entry") == entry_id:
                return x
        return None

    def finish_counts(self, st: State, entry_id: int, env: Env, ind: str, out: list, host: bool) -> None:
        """A scope finishing (_finish_scope): exit edges with `accesses`
        count it once; the others summed their commits already."""
        if self.rep is None:
            return
        x = self.exit_of(st, entry_id)
        if x is None:
            return
        for o in st.out_edges(x.id):
            m = o.memlet
            if m.is_empty or m.accesses is None:
                v = "0"
            else:
                v = env.emit(m.accesses)
            if host:
                self.hcount(self.ekey(st, o), v, out)
            else:
                self.dcount(self.ekey(st, o), v, ind, out)

    # -- custom write-conflict resolution --------------------------------------

    def wcr_fn(self, m, basetype: str) -> str:
        """Name of the combine function for memlet ``m``: a built-in one, or a
        __device__ function translated from the custom WCR's tasklet
        (ir.py:100-121: ``out = f(old, new)``)."""
        if m.wcr in ("sum", "product", "min", "max"):
            return m.wcr
        if m.wcr != "custom" or not m.wcr_doc or "code" not in m.wcr_doc:
            raise LoweringError(f"WCR '{m.wcr}' is not lowered")
        doc = m.wcr_doc
        key = (doc["code"], tuple(doc["inputs"]), tuple(doc["outputs"]), basetype)
        if key not in self.custom_wcr:
            old, new = doc["inputs"]
            out = doc["outputs"][0]
            name = f"custom{len(self.custom_wcr)}"
            types = {old: basetype, new: basetype, out: basetype}
            names = {old: "a_old", new: "a_new", out: "r_out"}
            tc = TaskletC(ast.parse(doc["code"]).body, types, names, {}, {}, {out}, set())
            t = CT[basetype]
            body = "\n".join(tc.emit("    "))
            self.devfns.insert(0, f"GEN_HD {t} wcr_{name}_f({t} a_old, {t} a_new) {{\n    {t} r_out = 0;\n"
                                  f"{body}\n    return r_out;\n}}\n"
                                  f"GEN_DEV void wcr_{name}({t}* p, {t} v) {{ wcr_cas(p, v, [](const {t} a, const {t} b) "
                                  f"{{ return wcr_{name}_f(a, b); }}); }}\n"
                                  f"GEN_HD void pwcr_{name}({t}* p, {t} v) {{ *p = wcr_{name}_f(*p, v); }}\n"
                                  f"#define GEN_WR_{name} 1\n"
                                  f"template <typename T> GEN_DEV void g_wr_{name}(T* p, int64_t i, int64_t n, T v, "
                                  f"int* err) {{ if (i < 0 || i >= n) {{ gen_fail(err, 1); return; }} wcr_{name}(p + i, v); }}\n"
                                  f"template <typename T> GEN_DEV void g_wr_p{name}(T* p, int64_t i, int64_t n, T v, "
                                  f"int* err) {{ if (i < 0 || i >= n) {{ gen_fail(err, 1); return; }} pwcr_{name}(p + i, v); }}\n")
            self.custom_wcr[key] = name
        return self.custom_wcr[key]

    # -- write targets --------------------------------------------------------

    def targets(self, st: State, e) -> list:
        """Access nodes behind a tasklet output edge, through scope exits;
        the committed memlet is the tasklet-side one (codegen.py:286-302)."""
        dst = st.nodes[e.dst]
        if dst.kind == "access":
            d = self.g.data.get(dst.data)
            if d is not None and d.kind == "stream" and d.transient:
                # a scope-local stream drained through the scope exit into an
                # outer stream (LocalStream, library.py): its pushes are the
                # outer stream's pushes -- the order is unspecified either way
                fwd = [o for o in st.out_edges(dst.id)
                       if st.nodes[o.dst].kind in ("map_exit", "consume_exit") and o.dst_conn]
                if fwd:
                    out = []
                    for o in fwd:
                        out += self.targets(st, type(e)(o.id, e.src, e.src_conn, o.dst, o.dst_conn, e.memlet))
                    return out
            return [dst]
        if dst.kind in ("map_exit", "consume_exit"):
            conn = "OUT_" + e.dst_conn[3:]
            out = []
            for nxt in st.out_edges(dst.id):
                if nxt.src_conn == conn:
                    out += self.targets(st, type(e)(nxt.id, e.src, e.src_conn, nxt.dst, nxt.dst_conn, e.memlet))
            return out
        raise LoweringError(f"unsupported write path through a {dst.kind} node")

    # -- scope bodies (device code) --------------------------------------------

    def emit_scope(self, st: State, parent: dict, entry: Optional[int], env: Env, ind: str, out: list,
                   in_map: bool) -> None:
        for nid in st.topological_order():
            if parent[nid] != entry or nid == entry:
                continue
            n = st.nodes[nid]
            if n.kind == "tasklet":
                self.emit_tasklet(st, n, env, ind, out, in_map)
            elif n.kind == "map_entry":
                self.emit_inner_map(st, parent, n, env, ind, out)
            elif n.kind == "access":
                self.emit_access_device(st, n, env, ind, out)
            elif n.kind == "nested":
                self.emit_nested_call(st, n, env, ind, out)
            elif n.kind in ("map_exit", "consume_exit"):
                continue
            else:
                raise LoweringError(f"'{n.kind}' nodes are not lowered inside a map scope")

    def dyn_range_locals(self, st: State, n, env: Env, ind: str, out: list) -> Env:
        more = {}
        for e in st.in_edges(n.id):
            if e.dst_conn and not e.dst_conn.startswith("IN_") and not e.memlet.is_empty:
                v = f"r_{_ident(e.dst_conn)}_{n.id}"
                pt = [env.emit(r.begin) for r in e.memlet.subset]
                out.append(f"{ind}const int64_t {v} = (int64_t){self.cname(e.memlet.data)}"
                           f"[{self.flat(e.memlet.data, pt, env)}];")
                more[e.dst_conn] = v
        return env.child(more)

    def emit_inner_map(self, st: State, parent: dict, n, env: Env, ind: str, out: list) -> None:
        outer = env
        env = self.dyn_range_locals(st, n, env, ind, out)
        more = {}
        depth = 0
        for p, r in zip(n.params, n.ranges):
            v = f"p_{_ident(p)}_{n.id}"
            sub = env.child(more)
            b, e_, s = sub.emit(r.begin), sub.emit(r.end), sub.emit(r.stride)
            out.append(f"{ind}{'    ' * depth}for (int64_t {v} = {b}; ({s}) > 0 ? {v} <= {e_} : {v} >= {e_}; "
                       f"{v} += {s}) {{")
            more[p] = v
            depth += 1
        self.instance_counts(st, n, env.child(more), ind + "    " * depth, out)
        self.emit_scope(st, parent, n.id, env.child(more), ind + "    " * depth, out, True)
        for d in reversed(range(depth)):
            out.append(f"{ind}{'    ' * d}}}")
        self.finish_counts(st, n.id, outer, ind, out, host=False)

    def emit_access_device(self, st: State, n, env: Env, ind: str, out: list) -> None:
        """Region copies into an access node inside a scope (LocalStorage
        copies, nested-graph scalar moves): element loops per thread."""
        self.access_counts(st, n, env, ind, out, host=False)
        for e in sorted(st.in_edges(n.id), key=lambda e: e.id):
            src = st.nodes[e.src]
            if e.memlet.is_empty or src.kind in ("tasklet", "map_exit", "nested"):
                continue
            m = e.memlet
            if self.g.data[m.data].kind == "stream" or self.g.data[n.data].kind == "stream":
                raise LoweringError("stream moves inside a map scope are not lowered")
            dsub = m.subset if m.data == n.data else m.reindex
            ssub = m.subset if m.data != n.data else (m.reindex if src.kind == "access" and m.reindex else m.subset)
            sdata = m.data if m.data != n.data else (src.data if src.kind == "access" else m.data)
            if m.data == n.data and src.kind == "access":
                # memlet names the destination: the source region is the reindex
                sdata, ssub, dsub = src.data, (m.reindex or m.subset), m.subset
            if dsub is None:
                raise LoweringError(f"copy into '{n.data}' lacks destination indices")
            self._copy_loops(sdata, ssub, n.data, dsub, env, ind, out)

    def _copy_loops(self, sdata, ssub, ddata, dsub, env: Env, ind: str, out: list) -> None:
        vs = []
        for k, r in enumerate(ssub):
            v = f"q{self.tcount}_{k}"
            vs.append(v)
            out.append(f"{ind}{'    ' * k}for (int64_t {v} = 0; {v} < g_rlen({env.emit(r.begin)}, "
                       f"{env.emit(r.end)}, 1); ++{v}) {{")
        self.tcount += 1
        deep = ind + "    " * len(vs)
        sidx = [f"({env.emit(r.begin)}) + {v}" for r, v in zip(ssub, vs)]
        if len(dsub) != len(ssub):
            # different ranks: copy in flat element order of the source region
            lin = vs[0]
            for k in range(1, len(vs)):
                lin = f"(({lin}) * g_rlen({env.emit(ssub[k].begin)}, {env.emit(ssub[k].end)}, 1) + {vs[k]})"
            didx = self.flat(ddata, [env.emit(r.begin) for r in dsub], env) + f" + ({lin})"
            out.append(f"{deep}{self.cname(ddata)}[{didx}] = {self.cname(sdata)}[{self.flat(sdata, sidx, env)}];")
        else:
            didx = [f"({env.emit(r.begin)}) + {v}" for r, v in zip(dsub, vs)]
            out.append(f"{deep}{self.cname(ddata)}[{self.flat(ddata, didx, env)}] = "
                       f"{self.cname(sdata)}[{self.flat(sdata, sidx, env)}];")
        for k in reversed(range(len(vs))):
            out.append(f"{ind}{'    ' * k}}}")

    def emit_tasklet(self, st: State, n, env: Env, ind: str, out: list, in_map: bool) -> None:
        code = n.code_ast
        prog_ins = list(n.doc.get("inputs", []))
        prog_outs = list(n.doc.get("outputs", []))
        reads, writes = _subscripts(code)
        t = self.tcount
        self.tcount += 1
        # Vectorization (library.py:763-840): memlets with a vector tile on
        # their last dimension; the body runs once per lane (codegen.py:408-444)
        width = 1
        for e in list(st.in_edges(n.id)) + list(st.out_edges(n.id)):
            if e.memlet.is_empty or not e.memlet.subset:
                continue
            tile = e.memlet.subset[-1].tile
            if not _is_one(tile):
                try:
                    w = int(X.evaluate(tile, {}))
                except X.ExprError as exc:
                    raise LoweringError(f"tasklet '{n.name}': symbolic vector width") from exc
                if width not in (1, w):
                    raise LoweringError(f"tasklet '{n.name}': mixed vector widths {width} and {w}")
                width = w
        lane = f"lv{t}"
        if self.rep is not None:
            # per firing: the invocation, and every output edge with `accesses`
            self.dcount("__tasklets", "1", ind, out)
            for e in st.out_edges(n.id):
                m = e.memlet
                if m.is_empty:
                    self.dcount(self.ekey(st, e), "0", ind, out)
                elif m.accesses is not None:
                    self.dcount(self.ekey(st, e), env.emit(m.accesses), ind, out)

        def point(sub):
            pt = [env.emit(r.begin) for r in sub]
            if width > 1 and not _is_one(sub[-1].tile):
                pt[-1] = f"({pt[-1]}) + {lane}"
            return pt
        if width > 1:
            out.append(f"{ind}for (int64_t {lane} = 0; {lane} < {width}; ++{lane}) {{")
            ind = ind + "    "
        out.append(f"{ind}{{  /* tasklet {n.name} */")
        ind2 = ind + "    "
        types, names, aread, awrite, dynamic = {}, {}, {}, {}, set()
        for e in st.in_edges(n.id):
            if e.memlet.is_empty or e.dst_conn is None:
                continue
            c, m = e.dst_conn, e.memlet
            d = self.g.data[m.data]
            types[c] = d.basetype
            if d.kind == "stream":
                if st.nodes[e.src].kind == "consume_entry" and m.data in self.pop_vars:
                    v = f"k{t}_{_ident(c)}"
                    out.append(f"{ind2}const {CT[d.basetype]} {v} = {self.pop_vars[m.data]};")
                    names[c] = v
                    continue
                raise LoweringError("stream pops outside a consume scope are not lowered")
            v = f"k{t}_{_ident(c)}"
            if c in reads:
                out.append(f"{ind2}const {CT[d.basetype]}* {v} = {self.cname(m.data)} + "
                           f"({self.origin(m.data, m.subset, env)});")
                # indexes run from the block origin through the container (codegen.py:417-420)
                aread[c] = (v, f"({self.size_expr(m.data, env)} - ({self.origin(m.data, m.subset, env)}))")
            else:
                pt = point(m.subset)
                self._track(m.data, m.subset, width)
                if self.unchecked:
                    out.append(f"{ind2}const {CT[d.basetype]} {v} = {self.cname(m.data)}[{self.flat(m.data, pt, env)}];")
                else:
                    out.append(f"{ind2}const {CT[d.basetype]} {v} = ({self.in_bounds(m.data, pt, env)}) ? "
                               f"{self.cname(m.data)}[{self.flat(m.data, pt, env)}] : "
                               f"(gen_fail(g_err, 6), ({CT[d.basetype]})0);")
            names[c] = v
        commits = []
        wcounts = []  # (edge, C count of subscript writes) for the report
        for e in st.out_edges(n.id):
            if e.memlet.is_empty or e.src_conn is None:
                continue
            c, m = e.src_conn, e.memlet
            tg = self.targets(st, e)
            if not tg:
                continue
            td = self.g.data[tg[0].data]
            types[c] = td.basetype
            v = f"k{t}_{_ident(c)}"
            names[c] = v
            if c in writes:
                fn = None if m.wcr is None else self.wcr_fn(m, td.basetype)
                priv = tg[0].data in self.private
                out.append(f"{ind2}{CT[td.basetype]}* {v} = {self.cname(tg[0].data)};")
                awrite[c] = (v, self.size_expr(tg[0].data, env), fn, priv)
                if self.rep is not None:
                    out.append(f"{ind2}int64_t {v}__nw = 0;")
                    wcounts.append((e, f"{v}__nw"))
                continue
            out.append(f"{ind2}{CT[td.basetype]} {v} = 0;")
            if m.is_dynamic:
                out.append(f"{ind2}int {v}__set = 0;")
                dynamic.add(c)
            commits.append((c, v, m, tg))
        for c in prog_outs:
            if c not in names:  # output without a memlet: a scratch local
                names[c] = f"k{t}_{_ident(c)}"
                types.setdefault(c, "float64")
                out.append(f"{ind2}{CT[types[c]]} {names[c]} = 0;")
        for c in prog_ins:
            if c not in names:
                raise LoweringError(f"tasklet '{n.name}': input '{c}' has no memlet")
        tc = TaskletC(code.body, types, names, aread, awrite, set(prog_outs), dynamic)
        tc.wcount = {e.src_conn: cv for e, cv in wcounts}
        out.extend(tc.emit(ind2))
        if self.rep is not None:
            # actual elements per lane: one per assigned scalar, one per
            # subscript write; the same amount crosses every exit behind it
            for c, v, m, tg in commits:
                e = next(x for x in st.out_edges(n.id) if x.src_conn == c and x.memlet is m)
                act = f"{v}__set" if m.is_dynamic else "1"
                if m.accesses is None:
                    self.dcount(self.ekey(st, e), act, ind2, out)
                self.chain_counts(st, e, act, ind2, out)
            for e, cv in wcounts:
                if e.memlet.accesses is None:
                    self.dcount(self.ekey(st, e), cv, ind2, out)
                self.chain_counts(st, e, cv, ind2, out)
        for c, v, m, tg in commits:
            for target in tg:
                td = self.g.data[target.data]
                guard = f"if ({v}__set) " if m.is_dynamic else ""
                if td.kind == "stream":
                    s = _ident(target.data)
                    if target.data in self.consumed:
                        out.append(f"{ind2}{guard}stream_push_q({self.cname(target.data)}, n_{s}, cap_{s}, r_{s}, "
                                   f"q_{s}, {v}, g_err);")
                    else:
                        out.append(f"{ind2}{guard}stream_push({self.cname(target.data)}, n_{s}, cap_{s}, {v}, g_err);")
                    continue
                sub = m.subset if m.data == target.data or m.reindex is None else m.reindex
                pt = point(sub)
                lv = f"{self.cname(target.data)}[{self.flat(target.data, pt, env)}]"
                self._track(target.data, sub, width)
                if not self.unchecked:
                    ok = self.in_bounds(target.data, pt, env)
                    guard = f"{guard}if (!({ok})) gen_fail(g_err, 6); else "
                if m.wcr is None:
                    out.append(f"{ind2}{guard}{lv} = {v};")
                else:
                    fn = self.wcr_fn(m, td.basetype)
                    priv = target.data in self.private
                    out.append(f"{ind2}{guard}{'p' if priv else ''}wcr_{fn}(&{lv}, ({CT[td.basetype]})({v}));")
        out.append(f"{ind}}}")
        if width > 1:
            out.append(f"{ind[:-4]}}}")

    # -- nested graphs ----------------------------------------------------------

    def emit_nested_call(self, st: State, n, env: Env, ind: str, out: list) -> None:
        inner = from_json(n.doc["sdfg"])
        fn = f"{self.prefix}_nested{len(self.devfns)}_{_ident(inner.name)}"
        sub = Lowering(inner, fn, nested=True, report=self.rep, keyprefix=f"{self.keyprefix}{inner.name}/")
        self.devfns.append(sub.device_function(fn))
        self.devfns[0:0] = sub.devfns  # deeper nests first
        bound = {}
        for e in list(st.in_edges(n.id)) + list(st.out_edges(n.id)):
            if e.memlet.is_empty:
                continue
            conn = e.dst_conn if e.dst == n.id else e.src_conn
            if conn in bound:
                continue
            bound[conn] = f"{self.cname(e.memlet.data)} + ({self.origin(e.memlet.data, e.memlet.subset, env)})"
        args = []
        for name, d in inner.data.items():
            if d.transient:
                continue
            if name not in bound:
                raise LoweringError(f"nested container '{name}' is not bound to an edge")
            args.append(bound[name])
        mapping = n.doc.get("symbol_mapping", {})
        for s in inner.symbols:
            if s not in mapping:
                raise LoweringError(f"nested symbol '{s}' is not mapped")
            args.append(env.emit(X.parse_expr(mapping[s])))
        args.append("g_err")
        if self.rep is not None:
            args.append("g_rep")
        out.append(f"{ind}{fn}({', '.join(args)});")
        for e in st.out_edges(n.id):  # _fire_nested: accesses or nothing
            m = e.memlet
            self.dcount(self.ekey(st, e), "0" if m.is_empty or m.accesses is None else env.emit(m.accesses), ind, out)

    def device_function(self, fn: str) -> str:
        """The nested graph as a __device__ function: private transients,
        a goto state machine over its states (codegen.py:663-700 shape)."""
        g = self.g
        params = [f"{CT[d.basetype]}* {self.cname(name)}" for name, d in g.data.items()
                  if not d.transient and d.kind == "array"]
        params += [f"int64_t s_{_ident(s)}" for s in g.symbols]
        params.append("int* g_err")
        if self.rep is not None:
            params.append("unsigned long long* g_rep")
        body = []
        for name, d in g.data.items():
            if d.kind == "stream":
                raise LoweringError("streams inside nested graphs are not lowered")
            if d.transient:
                sz = self.static_size(d)
                if sz is None or sz > MAX_PRIVATE:
                    raise LoweringError(f"nested transient '{name}' needs a static size <= {MAX_PRIVATE}")
                body.append(f"    {CT[d.basetype]} {self.cname(name)}[{sz}] = {{}};")
                self.private.add(name)
        for s in self.sym_names[len(g.symbols):]:
            body.append(f"    int64_t s_{_ident(s)} = 0;")
        env = Env(self, {}, host=False)
        body.append(f"    goto st_{_ident(g.start_state)};")
        for st in g.states:
            body.append(f"st_{_ident(st.name)}:;")
            inner: list = []
            parent = st.scope_parent()
            self.emit_scope(st, parent, None, env, "    ", inner, False)
            body += inner
            body += self._dispatch(st.name, env, "    ", prefix="st_", end="st__end")
        body.append("st__end:;")
        return f"__device__ __noinline__ void {fn}({', '.join(params)}) {{\n" + "\n".join(body) + "\n}\n"

    def _dispatch(self, name: str, env: Env, ind: str, prefix: str, end: str) -> list:
        out = []
        for t in self.g.out_transitions(name):
            assigns = "".join(f" s_{_ident(a)} = {env.emit(v)};" for a, v in t.assignments)
            go = f"goto {prefix}{_ident(t.dst)};"
            if t.condition == X.Num(1):
                out.append(f"{ind}{{{assigns} {go} }}")
                return out
            out.append(f"{ind}if ({env.emit(t.condition)}) {{{assigns} {go} }}")
        out.append(f"{ind}goto {end};")
        return out

    # -- top level (host-driven) ---------------------------------------------------

    def new_kernel(self, body: list, tag: str) -> str:
        name = f"{self.prefix}_k{self.kcount}_{_ident(tag)}"
        self.kcount += 1
        wait = '    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the previous kernel is done'
        self.kernels.append(f"__global__ void __launch_bounds__(256) {name}({self.kparams()}) {{\n"
                            + "\n".join([wait] + body) + "\n}\n")
        return name

    def top_map(self, st: State, parent: dict, n, host_env: Env, out: list) -> None:
        dynamic = any(e.dst_conn and not e.dst_conn.startswith("IN_") and not e.memlet.is_empty
                      for e in st.in_edges(n.id))
        denv = Env(self, {}, host=False)
        body = []
        scoped = sorted(x for x, (sn, top) in self.scoped.items() if sn == st.name and top == n.id)
        for x in scoped:  # this thread's slice
            body.append(f"    {self.cname(x)} += (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * "
                        f"{self.size_expr(x, denv)};")
        if dynamic:
            # data-dependent range (e.g. the SpMV row map after MapToForLoop):
            # every thread reads the bounds from HBM, the grid is fixed
            denv = self.dyn_range_locals(st, n, denv, "    ", body)
        lens, begins, strides = [], [], []
        for k, r in enumerate(n.ranges):
            body.append(f"    const int64_t b{k} = {denv.emit(r.begin)}, s{k} = {denv.emit(r.stride)}, "
                        f"n{k} = g_rlen(b{k}, {denv.emit(r.end)}, s{k});")
            lens.append(f"n{k}")
        body.append(f"    const int64_t total = {' * '.join(lens)};")
        head = ["    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total; "
                "f += (int64_t)gridDim.x * blockDim.x) {", "        int64_t rem = f;"]
        more = {}
        for k in reversed(range(len(n.params))):
            v = f"p_{_ident(n.params[k])}_{n.id}"
            # the outermost index needs no modulo: rem < n0 once the inner ones are divided out
            idx = "rem" if k == 0 else f"(rem % n{k})"
            head.append(f"        const int64_t {v} = b{k} + {idx} * s{k};")
            if k:
                head.append(f"        rem /= n{k};")
            more[n.params[k]] = v
        penv = denv.child(more)
        loop = list(head)
        self.instance_counts(st, n, penv, "        ", loop)
        # private transients: fresh, zeroed per iteration
        owned = [name for name in sorted(self.private) if self._owned_by(name, st, parent, n.id)]
        for name in owned:
            d = self.g.data[name]
            loop.append(f"        {CT[d.basetype]} {self.cname(name)}[{self.static_size(d)}] = {{}};")
        hoist = (not dynamic and not scoped and not owned and self.rep is None
                 and all(st.nodes[i].kind in ("tasklet", "map_exit") for i in st.topological_order()
                         if parent[i] == n.id and i != n.id))
        inner: list = []
        self.track = [] if hoist else None
        self.emit_scope(st, parent, n.id, penv, "        ", inner, True)
        track, self.track = self.track, None
        safe = self._corner_checks(n, denv, track) if hoist else None
        if safe:
            # every access of the body is affine in the map parameters: its
            # extremes are at the corners of the iteration box, so one check
            # of the corners per thread replaces the per-access checks
            unchecked: list = []
            self.unchecked = True
            try:
                self.emit_scope(st, parent, n.id, penv, "        ", unchecked, True)
            finally:
                self.unchecked = False
            body.append(f"    const bool g_safe = {safe};")
            body.append("    if (g_safe) {")
            body += head + unchecked + ["    }", "    } else {"]
            body += loop + inner + ["    }", "    }"]
        else:
            body += loop + inner + ["    }"]
        k = self.new_kernel(body, f"{st.name}_map{n.id}")
        self.finish_counts(st, n.id, host_env, "    ", out, host=True)

        def grow(nth: str) -> None:
            for x in scoped:
                c, bt = self.cname(x), CT[self.g.data[x].basetype]
                out.append(f"      {{ const int64_t need = ({nth}) * {self.size_expr(x, host_env)};")
                out.append(f"        if (need > tcap_{_ident(x)}) {{ if ({c}) cudaFreeAsync({c}, st); {c} = nullptr;")
                out.append(f"          if (cudaMallocAsync((void**)&{c}, (size_t)need * sizeof({bt}), st) != "
                           f"cudaSuccess) goto gen_fail;")
                out.append(f"          cudaMemsetAsync({c}, 0, (size_t)need * sizeof({bt}), st); "
                           f"tcap_{_ident(x)} = need; }} }}")
        if dynamic:
            grow("148LL * 256")
            out.append(f"    {k}<<<148, 256, 0, st>>>({self.kargs()}); GEN_CHECK();")
            return
        # host: launch over the same flattened range
        tot = " * ".join(f"g_rlen({host_env.emit(r.begin)}, {host_env.emit(r.end)}, {host_env.emit(r.stride)})"
                         for r in n.ranges)
        out.append(f"    {{ const int64_t tot = {tot};")
        out.append("      if (tot > 0) {")
        grow("(int64_t)gen_blocks(tot) * 256")
        args = self.kargs()
        out.append(f"      gen_launch({k}, gen_blocks(tot), 256, st{', ' + args if args else ''}); GEN_CHECK(); }} }}")

    def _corner_checks(self, n, denv: Env, track) -> Optional[str]:
        """The in-bounds condition of every recorded access at every corner
        of the map's iteration box (params at their first / last value), or
        None when an access is not affine in the parameters."""
        from itertools import product
        params = list(n.params)
        pset = set(params)
        if not track or any(t is None or not all(_affine_in(b, pset) for b in t[1]) for t in track):
            return None
        conds = []
        for combo in product((0, 1), repeat=len(params)):
            cenv = denv.child({p: (f"(b{k})" if c == 0 else f"(b{k} + (n{k} - 1) * s{k})")
                               for k, (p, c) in enumerate(zip(params, combo))})
            for data, begins in track:
                c = self.in_bounds(data, [cenv.emit(b) for b in begins], cenv)
                if c not in conds:
                    conds.append(c)
        return " && ".join(f"({c})" for c in conds)

    def top_consume(self, st: State, parent: dict, n, out: list) -> None:
        """A consume scope (codegen.py:526-543: P workers popping until the
        quiescence condition fails) as a persistent work-queue kernel.
        Every resident thread is a worker: it takes a ticket, waits for that
        item or for quiescence (every pushed item finished and nothing left
        to pop), runs the scope body on the item, and counts it finished
        after the body's pushes.  Only ``size(S) > 0`` conditions -- run
        until the stream is drained -- are lowered."""
        if any(sn == st.name and top == n.id for sn, top in self.scoped.values()):
            raise LoweringError("a consume scope's transients need a static size")
        se = next((e for e in st.in_edges(n.id) if e.dst_conn == "IN_stream"), None)
        if se is None or se.memlet.is_empty:
            raise LoweringError("consume entry without a stream")
        S = se.memlet.data
        cond = X.parse_expr(n.doc["condition"])
        ok = (isinstance(cond, X.Cmp) and isinstance(cond.left, X.Call) and cond.left.fn == "size"
              and cond.left.args[0] == X.Sym(S) and
              ((cond.op == ">" and cond.right == X.Num(0)) or (cond.op == ">=" and cond.right == X.Num(1))))
        if not ok:
            raise LoweringError(f"consume condition '{n.doc['condition']}' is not 'size({S}) > 0'")
        s = _ident(S)
        bt = CT[self.g.data[S].basetype]
        denv = Env(self, {}, host=False)
        self.pop_vars[S] = "elem"
        body = ["    const int64_t wid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;",
                "    for (;;) {",
                f"        const unsigned long long h = atomicAdd(&q_{s}[0], 1ull);",
                "        bool got = false;",
                "        for (long long spin = 0;; ++spin) {",
                f"            if ((int64_t)h < cap_{s} && ld_acq_u32(r_{s} + h)) {{ got = true; break; }}",
                f"            const unsigned long long F = ld_acq_u64(&q_{s}[1]);",
                f"            const unsigned long long T = ld_acq_u64(n_{s});",
                "            if (F == T && h >= T) break;",
                "            if (*(volatile int*)g_err) return;",
                "            if (spin > (1LL << 26)) { gen_fail(g_err, 5); return; }  // watchdog (~seconds)",
                "            __nanosleep(64);",
                "        }",
                "        if (!got) return;",
                f"        const {bt} elem = {self.cname(S)}[h];"]
        penv = denv.child({n.doc["param"]: f"(wid % g_imax(1LL, {denv.emit(X.parse_expr(n.doc['num_pes']))}))"})
        inner: list = []
        self.dcount(self.ekey(st, se), "1", "        ", inner)  # popped (interpreter.py:595)
        self.instance_counts(st, n, penv, "        ", inner)
        self.emit_scope(st, parent, n.id, penv, "        ", inner, True)
        body += inner
        body += ["        __threadfence();", f"        atomicAdd(&q_{s}[1], 1ull);", "    }"]
        del self.pop_vars[S]
        k = self.new_kernel(body, f"{st.name}_consume{n.id}")
        self.finish_counts(st, n.id, Env(self, {}, host=True), "    ", out, host=True)
        out.append(f"    {k}<<<148 * 4, 128, 0, st>>>({self.kargs()}); GEN_CHECK();")
        out.append(f"    gen_queue_reset<<<gen_blocks(cap_{s}), 256, 0, st>>>(r_{s}, n_{s}, q_{s}, cap_{s}); "
                   f"GEN_CHECK();")
        out.append(f"    cudaMemsetAsync(n_{s}, 0, 8, st); cudaMemsetAsync(q_{s}, 0, 16, st); ub_{s} = 0;")

    def _owned_by(self, name: str, st: State, parent: dict, entry: int) -> bool:
        for n in st.nodes:
            if n.kind == "access" and n.data == name:
                top = parent[n.id]
                while top is not None and parent[top] is not None:
                    top = parent[top]
                return top == entry
        return False

    def top_single(self, st: State, parent: dict, n, out: list, kind: str) -> None:
        denv = Env(self, {}, host=False)
        body = ["    if (blockIdx.x != 0 || threadIdx.x != 0) return;"]
        inner: list = []
        if kind == "tasklet":
            self.emit_tasklet(st, n, denv, "    ", inner, False)
        else:
            self.emit_nested_call(st, n, denv, "    ", inner)
        body += inner
        k = self.new_kernel(body, f"{st.name}_{kind}{n.id}")
        out.append(f"    {k}<<<1, 32, 0, st>>>({self.kargs()}); GEN_CHECK();")

    def top_access(self, st: State, n, host_env: Env, out: list) -> None:
        d = self.g.data[n.data]
        for e in sorted(st.in_edges(n.id), key=lambda e: e.id):
            src = st.nodes[e.src]
            if e.memlet.is_empty or src.kind in ("tasklet", "map_exit", "consume_exit", "nested", "reduce"):
                continue
            m = e.memlet
            sdata = src.data if src.kind == "access" else m.data
            sd = self.g.data[sdata]
            if sd.kind == "stream":
                if d.kind == "stream":
                    raise LoweringError("stream-to-stream moves are not lowered")
                s = _ident(sdata)
                out.append(f"    gen_drain<<<gen_blocks(cap_{s}), 256, 0, st>>>({self.cname(sdata)}, n_{s}, "
                           f"{self.cname(n.data)}, {self.size_expr(n.data, host_env)}, g_err); GEN_CHECK();")
                if self.rep is not None and m.accesses is None:  # the items drained
                    out.append(f"    gen_rep_addp<<<1, 1, 0, st>>>(g_rep + {self.slot(self.ekey(st, e))}, n_{s}); "
                               f"GEN_CHECK();")
                out.append(f"    cudaMemsetAsync(n_{s}, 0, 8, st); ub_{s} = 0;")
                continue
            if d.kind == "stream":
                raise LoweringError("array-to-stream bulk pushes are not lowered")
            if m.data == n.data:
                dsub, ssub = m.subset, (m.reindex or m.subset)
            else:
                ssub, dsub = m.subset, m.reindex
            if dsub is None:
                raise LoweringError(f"copy into '{n.data}' lacks destination indices")
            denv = Env(self, {}, host=False)
            body = []
            lens = [f"g_rlen({denv.emit(r.begin)}, {denv.emit(r.end)}, 1)" for r in ssub]
            body.append(f"    const int64_t total = {' * '.join(lens)};")
            body.append("    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total; "
                        "f += (int64_t)gridDim.x * blockDim.x) {")
            body.append("        int64_t rem = f;")
            vs = [None] * len(ssub)
            for k in reversed(range(len(ssub))):
                body.append(f"        const int64_t i{k} = rem % ({lens[k]}); rem /= ({lens[k]});")
                vs[k] = f"i{k}"
            sidx = [f"({denv.emit(r.begin)}) + {v}" for r, v in zip(ssub, vs)]
            if len(dsub) == len(ssub):
                didx = self.flat(n.data, [f"({denv.emit(r.begin)}) + {v}" for r, v in zip(dsub, vs)], denv)
            else:
                didx = self.flat(n.data, [denv.emit(r.begin) for r in dsub], denv) + " + f"
            body.append(f"        {self.cname(n.data)}[{didx}] = {self.cname(sdata)}[{self.flat(sdata, sidx, denv)}];")
            body.append("    }")
            k = self.new_kernel(body, f"{st.name}_copy{e.id}")
            tot = " * ".join(f"g_rlen({host_env.emit(r.begin)}, {host_env.emit(r.end)}, 1)" for r in ssub)
            out.append(f"    {{ const int64_t tot = {tot}; if (tot > 0) {{ {k}<<<gen_blocks(tot), 256, 0, st>>>"
                       f"({self.kargs()}); GEN_CHECK(); }} }}")

    def top_reduce(self, st: State, n, host_env: Env, out: list) -> None:
        ine = next(e for e in st.in_edges(n.id) if e.dst_conn == "in")
        oute = next(e for e in st.out_edges(n.id) if e.src_conn == "out")
        tgt = self.targets(st, oute)[0]
        wdoc = n.doc.get("wcr") if isinstance(n.doc.get("wcr"), dict) else {"kind": n.doc.get("wcr")}
        kind = wdoc.get("kind")
        axes = [int(a) for a in n.doc.get("axes", [])]
        td = self.g.data[tgt.data]

        class _M:  # the reduce's resolution, shaped like a memlet for wcr_fn
            wcr, wcr_doc = kind, wdoc
        wcr = self.wcr_fn(_M, td.basetype)
        if kind == "custom":
            iv = float(wdoc["identity"])
            ident = repr(iv) if td.basetype == "float64" else f"{int(iv)}LL"
        else:
            ident = {("sum", "float64"): "0.0", ("sum", "int64"): "0LL", ("product", "float64"): "1.0",
                     ("product", "int64"): "1LL", ("min", "float64"): "INFINITY", ("max", "float64"): "-INFINITY",
                     ("min", "int64"): "INT64_MAX", ("max", "int64"): "INT64_MIN"}[(kind, td.basetype)]
        denv = Env(self, {}, host=False)
        tsub = oute.memlet.subset if oute.memlet.data == tgt.data else oute.memlet.reindex
        isub = ine.memlet.subset
        # identity init of the target region
        tl = [f"g_rlen({denv.emit(r.begin)}, {denv.emit(r.end)}, 1)" for r in tsub]
        b1 = [f"    const int64_t total = {' * '.join(tl)};",
              "    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total; "
              "f += (int64_t)gridDim.x * blockDim.x) {", "        int64_t rem = f;"]
        for k in reversed(range(len(tsub))):
            b1.append(f"        const int64_t i{k} = rem % ({tl[k]}); rem /= ({tl[k]});")
        tidx = self.flat(tgt.data, [f"({denv.emit(r.begin)}) + i{k}" for k, r in enumerate(tsub)], denv)
        b1 += [f"        {self.cname(tgt.data)}[{tidx}] = {ident};", "    }"]
        k1 = self.new_kernel(b1, f"{st.name}_reduce_init{n.id}")
        il = [f"g_rlen({denv.emit(r.begin)}, {denv.emit(r.end)}, 1)" for r in isub]
        b2 = [f"    const int64_t total = {' * '.join(il)};",
              "    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total; "
              "f += (int64_t)gridDim.x * blockDim.x) {", "        int64_t rem = f;"]
        for k in reversed(range(len(isub))):
            b2.append(f"        const int64_t j{k} = rem % ({il[k]}); rem /= ({il[k]});")
        kept = [k for k in range(len(isub)) if k not in axes]
        oidx = self.flat(tgt.data, [f"({denv.emit(tsub[p].begin)}) + j{k}" for p, k in enumerate(kept)], denv)
        sidx = self.flat(ine.memlet.data, [f"({denv.emit(r.begin)}) + j{k}" for k, r in enumerate(isub)], denv)
        b2 += [f"        wcr_{wcr}(&{self.cname(tgt.data)}[{oidx}], {self.cname(ine.memlet.data)}[{sidx}]);",
               "    }"]
        k2 = self.new_kernel(b2, f"{st.name}_reduce{n.id}")
        htl = " * ".join(f"g_rlen({host_env.emit(r.begin)}, {host_env.emit(r.end)}, 1)" for r in tsub)
        hil = " * ".join(f"g_rlen({host_env.emit(r.begin)}, {host_env.emit(r.end)}, 1)" for r in isub)
        out.append(f"    {k1}<<<gen_blocks({htl}), 256, 0, st>>>({self.kargs()}); GEN_CHECK();")
        if self.rep is not None:  # _fire_reduce produces the reduced block
            kl = [f"g_rlen({host_env.emit(r.begin)}, {host_env.emit(r.end)}, {host_env.emit(r.stride)})"
                  for k, r in enumerate(isub) if k not in axes]
            m = oute.memlet
            v = host_env.emit(m.accesses) if m.accesses is not None else ("(" + " * ".join(kl) + ")" if kl else "1LL")
            self.hcount(self.ekey(st, oute), v, out)
        out.append(f"    {k2}<<<gen_blocks({hil}), 256, 0, st>>>({self.kargs()}); GEN_CHECK();")

    def stream_pushes(self, st: State, parent: dict, host_env: Env) -> dict:
        """Upper bound of pushes per stream in one execution of the state:
        trip count of the map nest around every pushing tasklet."""
        need: dict[str, list] = {}
        for n in st.nodes:
            if n.kind != "tasklet":
                continue
            for e in st.out_edges(n.id):
                if e.memlet.is_empty:
                    continue
                for tg in self.targets(st, e):
                    if self.g.data[tg.data].kind != "stream":
                        continue
                    trips = []
                    p = parent[n.id]
                    while p is not None:
                        me = st.nodes[p]
                        for r in me.ranges:
                            try:
                                trips.append(f"g_rlen({host_env.emit(r.begin)}, {host_env.emit(r.end)}, "
                                             f"{host_env.emit(r.stride)})")
                            except LoweringError as exc:
                                raise LoweringError(f"push into '{tg.data}' under a data-dependent range: "
                                                    f"{exc}") from exc
                        p = parent[p]
                    need.setdefault(tg.data, []).append(" * ".join(trips) if trips else "1")
        return need

    def program(self) -> Lowered:
        g = self.g
        henv = Env(self, {}, host=True)
        ptr_args = g.pointer_args()
        rsig = (", unsigned long long* g_reph, int64_t* g_vis, int64_t g_vcap, int64_t* g_nvis"
                if self.rep is not None else "")
        lines = ["extern \"C\" int " + self.prefix + "_run(void** ptrs, const int64_t* syms, void* stream_, "
                 "int* status" + rsig + ") {",
                 "    cudaStream_t st = (cudaStream_t)stream_;",
                 "    gen_pool_keep();",
                 "    cudaError_t gen_ce = cudaSuccess;",
                 "#define GEN_CHECK() do { gen_ce = cudaGetLastError(); if (gen_ce != cudaSuccess) goto gen_fail; } while (0)"]
        for i, (name, bt) in enumerate(ptr_args):
            lines.append(f"    {CT[bt]}* {self.cname(name)} = ({CT[bt]}*)ptrs[{i}];")
        for i, s in enumerate(g.symbols):
            lines.append(f"    int64_t s_{_ident(s)} = syms[{i}];")
        for s in self.sym_names[len(g.symbols):]:
            lines.append(f"    int64_t s_{_ident(s)} = 0;")
        lines.append("    int* g_err = nullptr;")
        if self.rep is not None:
            lines += ["    unsigned long long* g_rep = nullptr;", "    int64_t g_nv = 0;"]
        trans = [(n, d) for n, d in g.data.items() if d.transient and d.kind == "array" and n not in self.private
                 and n not in self.scoped]
        for name in sorted(self.scoped):
            lines += [f"    {CT[g.data[name].basetype]}* {self.cname(name)} = nullptr;",
                      f"    int64_t tcap_{_ident(name)} = 0;"]
        streams = [(n, d) for n, d in g.data.items() if d.kind == "stream"]
        for name, d in trans:
            lines.append(f"    {CT[d.basetype]}* {self.cname(name)} = nullptr;")
        for name, d in streams:
            s = _ident(name)
            if self.static_size(d) != 1:
                raise LoweringError(f"stream '{name}': only single-queue streams are lowered")
            lines += [f"    {CT[d.basetype]}* {self.cname(name)} = nullptr;",
                      f"    unsigned long long* n_{s} = nullptr;",
                      f"    int64_t cap_{s} = 0, ub_{s} = 0;"]
            if name in self.consumed:
                lines += [f"    unsigned* r_{s} = nullptr;", f"    unsigned long long* q_{s} = nullptr;"]
        lines.append("    int* g_status = gen_status_host();")
        lines.append("    g_err = gen_err_dev();")
        lines.append("    if (!g_err || !g_status) return 2;")
        lines.append("    cudaMemsetAsync(g_err, 0, 16, st);")
        if self.rep is not None:
            lines.append("    if (cudaMallocAsync((void**)&g_rep, @NREP@ * 8, st) != cudaSuccess) goto gen_fail;")
            lines.append("    cudaMemsetAsync(g_rep, 0, @NREP@ * 8, st);")
        for name, d in trans:
            lines.append(f"    {{ const size_t nb = (size_t)({self.size_expr(name, henv)}) * sizeof({CT[d.basetype]});")
            lines.append(f"      if (cudaMallocAsync((void**)&{self.cname(name)}, nb ? nb : 8, st) != cudaSuccess) "
                         f"goto gen_fail; cudaMemsetAsync({self.cname(name)}, 0, nb, st); }}")
        for name, d in streams:
            s = _ident(name)
            lines.append(f"    if (cudaMallocAsync((void**)&n_{s}, 8, st) != cudaSuccess) goto gen_fail;")
            lines.append(f"    cudaMemsetAsync(n_{s}, 0, 8, st);")
            if name in self.consumed:
                bt = CT[d.basetype]
                lines.append(f"    cap_{s} = {QUEUE_ITEMS}LL;")
                lines.append(f"    if (cudaMallocAsync((void**)&{self.cname(name)}, (size_t)cap_{s} * sizeof({bt}), st) "
                             f"!= cudaSuccess || cudaMallocAsync((void**)&r_{s}, (size_t)cap_{s} * 4, st) != cudaSuccess "
                             f"|| cudaMallocAsync((void**)&q_{s}, 16, st) != cudaSuccess) goto gen_fail;")
                lines.append(f"    cudaMemsetAsync(r_{s}, 0, (size_t)cap_{s} * 4, st); cudaMemsetAsync(q_{s}, 0, 16, st);")
        lines.append(f"    goto st_{_ident(g.start_state)};")
        for st in g.states:
            parent = st.scope_parent()
            lines.append(f"st_{_ident(st.name)}:;")
            lines.append("    {")
            if self.rep is not None:
                lines.append(f"    if (g_nv < g_vcap) g_vis[g_nv] = {g.states.index(st)}; ++g_nv;")
            for sname, trips in self.stream_pushes(st, parent, henv).items():
                if sname in self.consumed:
                    continue  # fixed-capacity work queue
                s = _ident(sname)
                bt = CT[g.data[sname].basetype]
                lines.append(f"    {{ const int64_t need = ub_{s} + {' + '.join(f'({t})' for t in trips)};")
                lines.append(f"      if (need > cap_{s}) {{ {bt}* nb = nullptr;")
                lines.append(f"        if (cudaMallocAsync((void**)&nb, (size_t)need * sizeof({bt}), st) != cudaSuccess) "
                             f"goto gen_fail;")
                lines.append(f"        if (cap_{s}) {{ cudaMemcpyAsync(nb, {self.cname(sname)}, (size_t)cap_{s} * "
                             f"sizeof({bt}), cudaMemcpyDeviceToDevice, st); cudaFreeAsync({self.cname(sname)}, st); }}")
                lines.append(f"        {self.cname(sname)} = nb; cap_{s} = need; }}")
                lines.append(f"      ub_{s} = need; }}")
            for nid in st.topological_order():
                if parent[nid] is not None:
                    continue
                n = st.nodes[nid]
                if n.kind == "map_entry":
                    self.top_map(st, parent, n, henv, lines)
                elif n.kind == "tasklet":
                    self.top_single(st, parent, n, lines, "tasklet")
                elif n.kind == "nested":
                    self.top_single(st, parent, n, lines, "nested")
                elif n.kind == "access":
                    self.top_access(st, n, henv, lines)
                    self.access_counts(st, n, henv, "    ", lines, host=True)
                elif n.kind == "reduce":
                    self.top_reduce(st, n, henv, lines)
                elif n.kind == "consume_entry":
                    self.top_consume(st, parent, n, lines)
                elif n.kind in ("map_exit", "consume_exit"):
                    continue
                else:
                    raise LoweringError(f"'{n.kind}' nodes are not lowered")
            lines.append("    }")
            lines += self._dispatch(st.name, henv, "    ", prefix="st_", end="st__end")
        lines.append("st__end:;")
        lines.append("    cudaMemcpyAsync(g_status, g_err, sizeof(int), cudaMemcpyDeviceToHost, st);")
        lines.append("    gen_ce = cudaStreamSynchronize(st);")
        lines.append("    if (gen_ce != cudaSuccess) goto gen_fail;")
        lines.append("    *status = *g_status;")
        if self.rep is not None:
            lines += ["    {", "    unsigned long long dv[@NREP@];",
                      "    gen_ce = cudaMemcpy(dv, g_rep, sizeof(dv), cudaMemcpyDeviceToHost);",
                      "    if (gen_ce != cudaSuccess) goto gen_fail;",
                      "    for (int i = 0; i < @NREP@; ++i) g_reph[i] += dv[i];",
                      "    *g_nvis = g_nv;", "    }", "    cudaFreeAsync(g_rep, st);"]
        free = [f"    if ({self.cname(n)}) cudaFreeAsync({self.cname(n)}, st);" for n, _ in trans]
        free += [f"    if ({self.cname(n)}) cudaFreeAsync({self.cname(n)}, st);" for n in sorted(self.scoped)]
        for name, _ in streams:
            free += [f"    if ({self.cname(name)}) cudaFreeAsync({self.cname(name)}, st);",
                     f"    if (n_{_ident(name)}) cudaFreeAsync(n_{_ident(name)}, st);"]
            if name in self.consumed:
                free += [f"    if (r_{_ident(name)}) cudaFreeAsync(r_{_ident(name)}, st);",
                         f"    if (q_{_ident(name)}) cudaFreeAsync(q_{_ident(name)}, st);"]
        lines += free  # stream-ordered: the outputs are already complete
        lines.append("    return 0;")
        lines.append("gen_fail:")
        lines += free
        if self.rep is not None:
            lines.append("    if (g_rep) cudaFreeAsync(g_rep, st);")
        lines.append("    cudaStreamSynchronize(st);")
        lines.append("    *status = -(int)gen_ce;")
        lines.append("    return 2;")
        lines.append("#undef GEN_CHECK")
        lines.append("}")
        keys = None
        if self.rep is not None:
            self.slot("__tasklets")
            keys = sorted(self.rep["slots"], key=self.rep["slots"].get)
            lines = [ln.replace("@NREP@", str(len(keys))) for ln in lines]
        host = "\n".join(lines)
        src = "\n".join([f"// generated by paper_1902_10345_b200.lower for SDFG '{g.name}'", PRELUDE,
                         SUBSCRIPT_HELPERS] + self.devfns + self.kernels + [host]) + "\n"
        digest = hashlib.sha256(src.encode()).hexdigest()[:16]
        return Lowered(g.name, src, f"{self.prefix}_run", ptr_args, list(g.symbols), digest,
                       report_keys=keys, state_names=[x.name for x in g.states] if keys is not None else None)


def _is_one(e) -> bool:
    return isinstance(e, X.Num) and e.value == 1


def _affine_in(e, params: set) -> bool:
    """e is affine in the symbols ``params`` (other symbols are uniform)."""
    if isinstance(e, (X.Num, X.Sym)):
        return True
    if isinstance(e, X.Neg):
        return _affine_in(e.arg, params)
    if isinstance(e, X.Bin) and e.op in ("+", "-"):
        return _affine_in(e.left, params) and _affine_in(e.right, params)
    if isinstance(e, X.Bin) and e.op == "*":
        lf, rf = X.free_symbols(e.left) & params, X.free_symbols(e.right) & params
        return (not lf and _affine_in(e.right, params)) or (not rf and _affine_in(e.left, params))
    return not (X.free_symbols(e) & params)


def _subscripts(code: ast.Module):
    reads, writes = set(), set()
    for node in ast.walk(code):
        if isinstance(node, ast.Assign):
            t = node.targets[0]
            if isinstance(t, ast.Subscript) and isinstance(t.value, ast.Name):
                writes.add(t.value.id)
        if isinstance(node, ast.Subscript) and isinstance(node.ctx, ast.Load) and isinstance(node.value, ast.Name):
            reads.add(node.value.id)
    return reads, writes


def lower(g: Graph, report: bool = False) -> Lowered:
    """``report=True``: the ExecutionReport build -- the same program with
    per-edge element counters and a state-visit log (slower: atomics)."""
    return Lowering(g, "gen_" + _ident(g.name), report={"slots": {}} if report else None).program()
