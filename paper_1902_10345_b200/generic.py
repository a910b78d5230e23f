"""Compile and run SDFGs through the generic Map/tasklet -> CUDA lowering
(lower.py): the B200 counterpart of the reference's ``generate`` +
``invoke_toolchain`` + ``CompiledSdfg.run`` (codegen.py:802-913) for graphs
that are not one of the five motif kernels.

The generated translation unit is compiled with nvcc for sm_100a into an
in-tree cache (``_gen/``, keyed by the source digest), loaded with ctypes,
and called with device pointers; containers keep the reference's basetypes
(float64/int64).  ``run`` has ``CompiledSdfg.run``'s contract: every
non-transient array is copied into a contiguous buffer of its declared
type, the program executes on the GPU, and the buffers come back.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import shutil
import subprocess
import threading
from typing import Any, Mapping

import numpy as np

from . import expr as X
from .errors import CodegenError, ExecutionError, OutOfBoundsError, ToolchainError
from .graph import Graph, load
from .lower import Lowered, lower

GEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_gen")
VISIT_LOG = 1 << 20  # state visits logged by report builds
_STATUS = {1: (OutOfBoundsError, "subscript write out of bounds"),
           2: (ExecutionError, "subscript read out of bounds"),
           3: (ExecutionError, "stream overflow"),
           4: (OutOfBoundsError, "stream drain overflows its target array"),
           5: (ExecutionError, "consume scope made no progress (watchdog)"),
           6: (OutOfBoundsError, "memlet index outside its container")}


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise ToolchainError("nvcc not found (the generic lowering compiles with nvcc for sm_100a)")


def build(lowered: Lowered) -> str:
    """nvcc -> _gen/<name>_<digest>.so (reused when present)."""
    os.makedirs(GEN_DIR, exist_ok=True)
    # -fmad=false: no a*b+c contraction, so float64 results match the
    # reference's gcc -O2 build and its interpreter bit for bit
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
             "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared"]
    key = hashlib.sha256((lowered.source + " ".join(flags)).encode()).hexdigest()[:16]
    base = os.path.join(GEN_DIR, f"{lowered.name}_{key}")
    so = base + ".so"
    if os.path.exists(so):
        return so
    # no lock around nvcc: concurrent builders of one key each compile to a
    # private temporary and the atomic rename makes the last one win
    tag = f"{os.getpid()}.{threading.get_ident()}"
    cu = f"{base}.{tag}.cu"
    with open(cu, "w") as f:
        f.write(lowered.source)
    tmp = f"{so}.{tag}.tmp"
    cmd = [nvcc()] + flags + ["-o", tmp, cu, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise ToolchainError(f"nvcc failed for '{lowered.name}':\n{r.stderr}")
    os.replace(cu, base + ".cu")
    os.replace(tmp, so)
    return so


class GenericProgram:
    """A lowered, compiled SDFG; ``run`` mirrors CompiledSdfg.run."""

    def __init__(self, g: Graph, lowered: Lowered, so_path: str):
        self.graph = g
        self.lowered = lowered
        self.path = so_path
        self._lib = ctypes.CDLL(so_path)
        self._fn = getattr(self._lib, lowered.entry)
        self._fn.restype = ctypes.c_int
        self._fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
        if lowered.report_keys is not None:  # counters + state-visit log
            self._fn.argtypes += [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]

    @property
    def reports(self) -> bool:
        return self.lowered.report_keys is not None

    @property
    def pointer_args(self):
        return self.lowered.pointer_args

    @property
    def symbol_args(self):
        return self.lowered.symbol_args

    def run(self, arrays: Mapping[str, Any], symbols: Mapping[str, int]) -> dict:
        return self._run(arrays, symbols)[0]

    def run_report(self, arrays: Mapping[str, Any], symbols: Mapping[str, int]) -> tuple:
        """``run`` plus the interpreter's ExecutionReport fields
        (interpreter.py:107-132) measured on the device: states_visited,
        elements_moved per memlet edge, total_moved, tasklet_invocations.
        Needs a report build (``compile_generic(g, report=True)``)."""
        if not self.reports:
            raise ExecutionError("this program was compiled without report counters")
        return self._run(arrays, symbols)

    def _report(self, counts, vis, nv: int) -> dict:
        keys = self.lowered.report_keys
        states = [self.lowered.state_names[i] for i in vis[:min(nv, len(vis))]]
        visited = set(states)
        moved = {}
        for k, c in zip(keys, counts):
            if k == "__tasklets":
                continue
            st = k.rsplit(":e", 1)[0]
            if c or ("/" not in st and st in visited):
                moved[k] = int(c)
        return {"states_visited": states, "elements_moved": dict(sorted(moved.items())),
                "total_moved": sum(moved.values()),
                "tasklet_invocations": int(counts[keys.index("__tasklets")])}

    def _run(self, arrays: Mapping[str, Any], symbols: Mapping[str, int]) -> tuple:
        import torch
        if not torch.cuda.is_available():
            raise ExecutionError("the generic B200 path needs a CUDA device")
        g = self.graph
        syms = {k: int(v) for k, v in symbols.items()}
        missing = [s for s in self.symbol_args if s not in syms]
        if missing:
            raise ExecutionError(f"unbound symbols: {sorted(missing)}")
        bufs, dev = {}, []
        for name, bt in self.pointer_args:
            if name not in arrays:
                raise ExecutionError(f"missing input container '{name}'")
            dt = np.int64 if bt == "int64" else np.float64
            buf = np.ascontiguousarray(np.asarray(arrays[name], dtype=dt)).copy()
            want = 1
            for d in g.data[name].dims:
                want *= int(X.evaluate(d, syms))
            if buf.size != want:
                raise ExecutionError(f"input '{name}' has {buf.size} elements; container expects {want}")
            bufs[name] = buf
            t = torch.from_numpy(buf.reshape(-1)).to("cuda") if buf.size else \
                torch.empty(1, dtype=torch.float64 if bt == "float64" else torch.int64, device="cuda")
            dev.append(t)
        ptrs = (ctypes.c_void_p * max(1, len(dev)))(*[t.data_ptr() for t in dev])
        svals = (ctypes.c_int64 * max(1, len(self.symbol_args)))(*[syms[s] for s in self.symbol_args])
        status = ctypes.c_int(0)
        stream = torch.cuda.current_stream().cuda_stream
        extra = []
        if self.reports:
            counts = np.zeros(len(self.lowered.report_keys), np.uint64)
            vis = np.zeros(VISIT_LOG, np.int64)
            nv = np.zeros(1, np.int64)
            extra = [counts.ctypes.data_as(ctypes.c_void_p), vis.ctypes.data_as(ctypes.c_void_p),
                     ctypes.c_int64(VISIT_LOG), nv.ctypes.data_as(ctypes.c_void_p)]
        rc = self._fn(ctypes.cast(ptrs, ctypes.c_void_p), ctypes.cast(svals, ctypes.c_void_p),
                      ctypes.c_void_p(stream), ctypes.byref(status), *extra)
        if rc != 0:
            raise ExecutionError(f"generic program '{g.name}' failed on the device (cuda status {-status.value})")
        if status.value:
            exc, msg = _STATUS.get(status.value, (ExecutionError, f"device error {status.value}"))
            raise exc(f"{msg} in '{g.name}'")
        for (name, _), t in zip(self.pointer_args, dev):
            if bufs[name].size:
                bufs[name].reshape(-1)[:] = t.cpu().numpy()
        return bufs, (self._report(counts, vis, int(nv[0])) if self.reports else None)


    def run_device(self, tensors: list, symbols: Mapping[str, int], stream=None) -> None:
        """Execute on device-resident containers (torch tensors in
        pointer_args order, contiguous, float64/int64): the timed path."""
        import torch
        syms = {k: int(v) for k, v in symbols.items()}
        if len(tensors) != len(self.pointer_args):
            raise ExecutionError(f"expected {len(self.pointer_args)} containers, got {len(tensors)}")
        for (name, bt), t in zip(self.pointer_args, tensors):
            want = torch.float64 if bt == "float64" else torch.int64
            if t.dtype != want or not t.is_cuda or not t.is_contiguous():
                raise ExecutionError(f"container '{name}' must be a contiguous CUDA {want} tensor")
        if self.reports:
            raise ExecutionError("run_device takes the timed build (compile_generic without report)")
        ptrs = (ctypes.c_void_p * max(1, len(tensors)))(*[t.data_ptr() for t in tensors])
        svals = (ctypes.c_int64 * max(1, len(self.symbol_args)))(*[syms[s] for s in self.symbol_args])
        status = ctypes.c_int(0)
        st = stream if stream is not None else torch.cuda.current_stream()
        rc = self._fn(ctypes.cast(ptrs, ctypes.c_void_p), ctypes.cast(svals, ctypes.c_void_p),
                      ctypes.c_void_p(st.cuda_stream), ctypes.byref(status))
        if rc != 0:
            raise ExecutionError(f"generic program '{self.graph.name}' failed on the device "
                                 f"(cuda status {-status.value})")
        if status.value:
            exc, msg = _STATUS.get(status.value, (ExecutionError, f"device error {status.value}"))
            raise exc(f"{msg} in '{self.graph.name}'")


def compile_generic(sdfg: Any, report: bool = False) -> GenericProgram:
    """Lower + nvcc + load.  CodegenError for constructs the lowering does
    not cover.  ``report=True`` builds the ExecutionReport variant."""
    g = load(sdfg)
    lw = lower(g, report=report)
    return GenericProgram(g, lw, build(lw))
