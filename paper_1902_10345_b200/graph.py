"""Read-only view of an SDFG in the reference's canonical interchange form.

The boundary between the reference toolkit and this backend is the
reference's own public JSON document (``sdfg.serialization.to_json``,
serialization.py:106-160; format ``sdfg.json`` version 1).  A reference
``Sdfg`` object is converted with that very function; a ``.sdfg.json`` file
or an already-loaded document is read directly.  This keeps the backend
importable where the reference is not installed (the GPU boxes) while the
structure and the names stay the reference's: states, access nodes,
tasklets, map entry/exit pairs, reduce nodes, memlets with WCR, streams,
and interstate transitions (ir.py:201-343, :651-702).
"""

from __future__ import annotations

import ast
import json
import os
import sys
from dataclasses import dataclass, field
from typing import Any, Optional

from .expr import Expr, Range, parse_expr, parse_range, parse_subset

FORMAT = "sdfg.json"


class GraphFormatError(ValueError):
    pass


@dataclass
class Desc:
    name: str
    basetype: str
    dims: tuple
    transient: bool
    kind: str
    storage: str


@dataclass
class Memlet:
    data: Optional[str]
    subset: Optional[tuple] = None
    reindex: Optional[tuple] = None
    accesses: Optional[Expr] = None
    wcr: Optional[str] = None
    wcr_doc: Optional[dict] = None  # custom WCR: code, inputs, outputs, identity (serialization.py:40-49)

    @property
    def is_empty(self) -> bool:
        return self.data is None

    @property
    def is_dynamic(self) -> bool:
        return not self.is_empty and self.accesses is None


@dataclass
class Node:
    id: int
    kind: str  # access | tasklet | map_entry | map_exit | reduce | consume_entry | ...
    doc: dict
    # parsed extras
    params: list = field(default_factory=list)
    ranges: list = field(default_factory=list)
    code_ast: Optional[ast.Module] = None

    @property
    def data(self):
        return self.doc.get("data")

    @property
    def name(self):
        return self.doc.get("name")


@dataclass
class Edge:
    id: int
    src: int
    src_conn: Optional[str]
    dst: int
    dst_conn: Optional[str]
    memlet: Memlet


@dataclass
class State:
    name: str
    nodes: list
    edges: list

    def in_edges(self, n: int):
        return [e for e in self.edges if e.dst == n]

    def out_edges(self, n: int):
        return [e for e in self.edges if e.src == n]

    def scope_parent(self) -> dict:
        """Innermost enclosing map entry of every node (ir.py:550-606 restated)."""
        order = self.topological_order()
        parent: dict[int, Optional[int]] = {}
        for v in order:
            node = self.nodes[v]
            cands = set()
            for e in self.in_edges(v):
                u = self.nodes[e.src]
                if u.kind in ("map_entry", "consume_entry"):
                    cands.add(u.id)
                elif u.kind in ("map_exit", "consume_exit"):
                    cands.add(parent[u.doc["entry"]])
                else:
                    cands.add(parent[u.id])
            if node.kind in ("map_exit", "consume_exit"):
                parent[v] = parent[node.doc["entry"]]
                continue
            if not cands:
                parent[v] = None
            elif len(cands) == 1:
                parent[v] = cands.pop()
            else:
                raise GraphFormatError(f"node {v} reached from conflicting scopes in '{self.name}'")
        return parent

    def topological_order(self) -> list:
        indeg = {n.id: 0 for n in self.nodes}
        for e in self.edges:
            indeg[e.dst] += 1
        ready = sorted(n for n, d in indeg.items() if d == 0)
        out = []
        while ready:
            n = ready.pop(0)
            out.append(n)
            for e in sorted(self.out_edges(n), key=lambda e: e.id):
                indeg[e.dst] -= 1
                if indeg[e.dst] == 0:
                    ready.append(e.dst)
            ready.sort()
        if len(out) != len(self.nodes):
            raise GraphFormatError(f"state '{self.name}' has a dataflow cycle")
        return out


@dataclass
class Transition:
    src: str
    dst: str
    condition: Expr
    assignments: list


@dataclass
class Graph:
    name: str
    symbols: list
    data: dict
    states: list
    start_state: str
    transitions: list
    doc: dict

    def state(self, name: str) -> Optional[State]:
        for s in self.states:
            if s.name == name:
                return s
        return None

    def out_transitions(self, name: str):
        return [t for t in self.transitions if t.src == name]

    def in_transitions(self, name: str):
        return [t for t in self.transitions if t.dst == name]

    def pointer_args(self) -> list:
        """Non-transient arrays in declaration order (codegen.py:620-627)."""
        return [(d.name, d.basetype) for d in self.data.values()
                if not d.transient and d.kind == "array"]


def _memlet(doc: dict) -> Memlet:
    if doc.get("empty"):
        return Memlet(None)
    return Memlet(
        data=doc["data"],
        subset=parse_subset(doc["subset"]),
        reindex=parse_subset(doc["reindex"]) if "reindex" in doc else None,
        accesses=parse_expr(doc["accesses"]) if "accesses" in doc else None,
        wcr=(doc.get("wcr") or {}).get("kind"),
        wcr_doc=doc.get("wcr"),
    )


def from_json(doc: dict) -> Graph:
    if doc.get("format") != FORMAT:
        raise GraphFormatError(f"not an {FORMAT} document (format={doc.get('format')!r})")
    data = {}
    for d in doc["data"]:
        data[d["name"]] = Desc(d["name"], d["basetype"], tuple(parse_expr(x) for x in d["dims"]),
                               bool(d["transient"]), d["kind"], d.get("storage", "heap"))
    states = []
    for s in doc["states"]:
        nodes = []
        for i, n in enumerate(s["nodes"]):
            node = Node(i, n["kind"], n)
            if n["kind"] == "map_entry":
                node.params = list(n["params"])
                node.ranges = [parse_range(r) for r in n["ranges"]]
            elif n["kind"] == "tasklet":
                node.code_ast = ast.parse(n["code"])
            nodes.append(node)
        edges = [Edge(i, e["src"], e["src_conn"], e["dst"], e["dst_conn"], _memlet(e["memlet"]))
                 for i, e in enumerate(s["edges"])]
        states.append(State(s["name"], nodes, edges))
    trans = [Transition(t["src"], t["dst"], parse_expr(t["condition"]),
                        [(k, parse_expr(v)) for k, v in t["assignments"]])
             for t in doc["transitions"]]
    return Graph(doc["name"], [s for s, _ in doc["symbols"]], data, states, doc["start_state"],
                 trans, doc)


def to_doc(obj: Any) -> dict:
    """Interchange document of ``obj``: a reference ``Sdfg`` (serialised with
    the reference's own ``to_json``), a JSON dict, a JSON string, or a path."""
    if isinstance(obj, dict):
        return obj
    if isinstance(obj, (str, os.PathLike)):
        s = str(obj)
        if os.path.exists(s):
            with open(s) as f:
                return json.load(f)
        return json.loads(s)
    if hasattr(obj, "states") and hasattr(obj, "data") and hasattr(obj, "symbols"):
        pkg = type(obj).__module__.rsplit(".", 1)[0]
        ser = sys.modules.get(pkg + ".serialization")
        if ser is None:
            import importlib
            ser = importlib.import_module(pkg + ".serialization")
        return ser.to_json(obj)
    raise GraphFormatError(f"cannot read an SDFG from {type(obj).__name__}")


def load(obj: Any) -> Graph:
    if isinstance(obj, Graph):
        return obj
    return from_json(to_doc(obj))
