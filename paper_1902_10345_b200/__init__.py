"""B200 (sm_100a) execution backend for SDFG Map scopes with write-conflict
resolution and stream memlets (arXiv 1902.10345 hot path).

Front door, mirroring the reference toolkit (/root/reference/pkg/src/sdfg):

    import paper_1902_10345_b200 as b200
    b200.register()                                   # adds GPUTransformMap to sdfg.rewriting
    m = find_matches(g, "GPUTransformMap")[0]
    g2, journal_entry = apply_transformation(g, m, {"precision": "fp32"})
    prog = b200.invoke_toolchain(b200.generate(g2))  # codegen.generate / invoke_toolchain
    outputs = prog.run(arrays, symbols)               # CompiledSdfg.run contract

The kernels live in libsdfgb200.so (C ABI: include/sdfgb200.h); see
DESIGN.md for the motif -> kernel map and INTEGRATION.md for the bindings.
"""

from .classify import Plan, UnsupportedGraph, classify  # noqa: F401
from .dispatch import (  # noqa: F401
    CompiledB200Sdfg,
    GeneratedB200Code,
    compile_b200,
    generate,
    invoke_toolchain,
)
from .errors import CodegenError, ExecutionError, OutOfBoundsError, ToolchainError  # noqa: F401
from .graph import load  # noqa: F401
from .transform import RULE_NAME, register, unregister  # noqa: F401

__version__ = "0.1.0"


def run(sdfg, arrays, symbols):
    """One-call execution of a GPU-marked SDFG; returns the output buffers."""
    return invoke_toolchain(generate(sdfg)).run(arrays, symbols)
