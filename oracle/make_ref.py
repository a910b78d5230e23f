"""Build ``oracle/_ref``: the reference's OWN CPU dispatcher output for each motif.

    python oracle/make_ref.py          (build container only: needs /root/reference)

The reference is a Python package whose CPU path *emits* C
(codegen.generate, codegen.py:802-848) and compiles it with
``cc -shared -fPIC -O2`` (codegen.invoke_toolchain, codegen.py:890-913).  This
script drives exactly those two public functions on the BASELINE-shaped motif
graphs (tests/golden/motifs_ref.py) with ``workdir=oracle/_ref``, so the
outputs are the reference's generated sources + shared objects, unmodified.
A manifest records each entry point's signature (GeneratedCode.pointer_args /
symbol_args, codegen.py:146-156) so the GPU box can call them through ctypes
without the reference installed.

Outputs go only to oracle/_ref/ (git-ignored, shipped to the GPU box).
The Jacobi graph is also emitted with the ``cpu_parallel`` schedule and built
with -fopenmp -- the reference's parallel CPU schedule (codegen.py:509-512);
it is race-free for Jacobi only.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(HERE, "_ref")
sys.path.insert(0, os.path.join(REPO, "tests", "golden"))


def main() -> int:
    import motifs_ref as M  # noqa: E402  (imports the reference)
    from sdfg.codegen import generate, invoke_toolchain  # noqa: E402
    from sdfg.ir import MapEntry  # noqa: E402

    os.makedirs(OUT, exist_ok=True)
    graphs = {
        "histogram": M.histogram(),
        "query": M.query("<"),
        "spmv": M.spmv(),
        "jacobi2d": M.jacobi2d(),
        "matmul": M.matmul(),
        # paper §5.2 chain (M1 CPU baseline)
        "matmul_chain32": M.matmul((("MapTiling", {"tile": 32}),
                                    ("LocalStorage", {"data": "B"}))),
    }
    graphs["matmul_chain32"].name = "matmul_chain32"
    jp = M.jacobi2d(name="jacobi2d_omp")
    for st in jp.states:
        for n in st.nodes.values():
            if isinstance(n, MapEntry):
                n.schedule = "cpu_parallel"
    graphs["jacobi2d_omp"] = jp
    # generic-lowering workloads (reference gallery, gallery.py:60-105, :498-545)
    from sdfg import gallery  # noqa: E402
    for name in ("laplace", "mandelbrot"):
        g = gallery.fixture(name).sdfg
        g.name = f"gal_{name}"
        graphs[f"gal_{name}"] = g
        go = gallery.fixture(name).sdfg
        go.name = f"gal_{name}_omp"
        for st in go.states:
            for n in st.nodes.values():
                if isinstance(n, MapEntry):
                    n.schedule = "cpu_parallel"
        graphs[f"gal_{name}_omp"] = go

    manifest = {}
    for key, g in graphs.items():
        code = generate(g)
        flags = ["-fopenmp"] if key.endswith("_omp") else None
        invoke_toolchain(code, flags=flags, workdir=OUT)
        manifest[key] = {
            "lib": f"lib{code.name}.so",
            "entry": code.name,
            "pointer_args": code.pointer_args,
            "symbol_args": code.symbol_args,
            "flags": (flags or []) + ["-shared", "-fPIC", "-O2"],
            "signature": code.signature(),
        }
        print(f"{key}: {code.signature()}")
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
