"""Motif recognition: which sm_100a kernel executes a given SDFG.

The reference dispatches a Map scope by walking it (interpreter
``_fire_map``, interpreter.py:547-562) or by emitting a C loop nest
(``emit_map``, codegen.py:500-524).  This backend instead recognises the
whole program as one of the hot-path motifs and binds it to a kernel.  The
recogniser is structural and semantic, not name-based:

* map nests are normalised first: tiled maps (MapTiling, library.py:557-594:
  outer ``p_t = b:e:s``, inner ``p = p_t:min(p_t + s - 1, e)``) and expanded
  maps (MapExpansion, library.py:258-323) flatten into one iteration domain;
  LocalStorage transients (library.py:644-722) are looked through by adding
  the copy's origin back onto the reindexed accesses;
* every tasklet input is resolved to ``container[affine index]`` over the
  flat parameters, and tasklet bodies are matched on their AST, so the
  arithmetic order the kernel must keep (tasklets.py:430-444) is read off
  the program, not assumed.

A program that matches no motif raises :class:`UnsupportedGraph` -- there is
no CPU fallback (north star: "no CPU fallback for those motifs").
"""

from __future__ import annotations

import ast
from dataclasses import dataclass, field
from typing import Optional

from . import expr as X
from .graph import Graph, Node, State

CMP_OPS = {ast.Lt: "<", ast.LtE: "<=", ast.Gt: ">", ast.GtE: ">=", ast.Eq: "==", ast.NotEq: "!="}
MIRROR = {"<": ">", "<=": ">=", ">": "<", ">=": "<=", "==": "==", "!=": "!="}


class UnsupportedGraph(ValueError):
    """No sm_100a motif kernel implements this program."""


@dataclass
class Plan:
    motif: str
    name: str
    pointer_args: list  # [(container, basetype)] in reference order (codegen.py:620-627)
    symbol_args: list  # reference symbol order
    roles: dict  # role -> container
    params: dict = field(default_factory=dict)
    main_state: str = ""
    main_map: int = -1
    dims: dict = field(default_factory=dict)  # container -> tuple(Expr)

    def shape(self, container: str, symbols: dict) -> tuple:
        return tuple(int(X.evaluate(d, symbols)) for d in self.dims[container])


# ----------------------------------------------------------------- helpers

def _top_maps(state: State, parent: dict) -> list:
    return [n for n in state.nodes if n.kind == "map_entry" and parent[n.id] is None]


def _exit_of(state: State, entry: Node) -> Node:
    for n in state.nodes:
        if n.kind == "map_exit" and n.doc["entry"] == entry.id:
            return n
    raise UnsupportedGraph(f"map {entry.id} has no exit")


def _children(parent: dict, eid: int) -> list:
    return [n for n, p in parent.items() if p == eid]


def _is_tile_end(end: X.Expr, tile_sym: str, step: int, outer_end: X.Expr) -> bool:
    """``min(tile_sym + step - 1, outer_end)`` in either argument order."""
    if not (isinstance(end, X.Call) and end.fn == "min" and len(end.args) == 2):
        return False
    for a, b in (end.args, end.args[::-1]):
        fa = X.affine(a)
        if fa is not None and fa.only(tile_sym) == step - 1 and X.same_value(b, outer_end):
            return True
    return False


@dataclass
class Nest:
    entries: list  # outer -> inner map entry nodes
    flat: dict  # param -> (begin Expr, end Expr), stride 1
    order: list  # flat params in nest order
    body: list  # node ids inside the innermost map (exits excluded)
    local: dict  # transient -> (container, origin exprs)   (LocalStorage)
    bind: dict = field(default_factory=dict)  # innermost name -> unique parameter name


def map_nest(state: State, top: Node, parent: dict) -> Nest:
    """Flatten the map nest under ``top``.  Parameters are renamed per level
    (``p#level``) because nested levels may legally shadow a name -- the
    reference's MapTiling picks ``p_t`` without looking at enclosing maps
    (library.py:576-580), and an inner binding wins (interpreter.py:559-560)."""
    entries = [top]
    local: dict = {}
    cur = top
    while True:
        kids = [state.nodes[k] for k in _children(parent, cur.id)]
        inner = [k for k in kids if k.kind == "map_entry"]
        rest = [k for k in kids if k.kind not in ("map_entry", "map_exit")]
        found: dict = {}
        if len(inner) == 1 and all(_is_local_storage(state, k, cur, inner[0], found) for k in rest):
            for k, (d, o) in found.items():
                local[k] = (d, o, len(entries) - 1)
            if _dynamic_connectors(inner[0]):
                break  # data-dependent inner range (spmv): not flattenable
            cur = inner[0]
            entries.append(cur)
            continue
        break
    body = [k for k in _children(parent, cur.id) if state.nodes[k].kind != "map_exit"]
    # flatten the iteration domain, resolving shadowed names level by level
    ranges = []
    bind: dict = {}
    snapshots = []
    for lvl, e in enumerate(entries):
        sub = {k: X.Sym(v) for k, v in bind.items()}
        rs = [X.Range(X.substitute(r.begin, sub), X.substitute(r.end, sub),
                      X.substitute(r.stride, sub), r.tile) for r in e.ranges]
        for p_ in e.params:
            bind[p_] = f"{p_}#{lvl}"
        snapshots.append(dict(bind))
        ranges.extend(zip([bind[p_] for p_ in e.params], rs))
    for k, (d, o, lvl) in list(local.items()):
        sub = {n: X.Sym(v) for n, v in snapshots[lvl].items()}
        local[k] = (d, tuple(X.substitute(x, sub) for x in o))
    flat: dict = {}
    order: list = []
    tiles: dict = {}
    used: set = set()
    for p, r in ranges:
        stride = X.evaluate(r.stride, {}) if not X.free_symbols(r.stride) else None
        if r.tile != X.Num(1):
            raise UnsupportedGraph(f"map parameter '{p}' has a tiled range")
        if stride is None or stride < 1:
            raise UnsupportedGraph(f"map parameter '{p}' has a non-constant stride")
        if stride != 1:
            tiles[p] = (r.begin, r.end, stride)
            continue
        b, e = r.begin, r.end
        # peel (possibly nested) MapTiling levels: p in [q : min(q + s - 1, E_q)]
        # with q in [B_q : E_q : s] covers exactly [B_q : E_q]
        while isinstance(b, X.Sym) and b.name in tiles:
            tb, te, ts = tiles[b.name]
            if not _is_tile_end(e, b.name, ts, te):
                raise UnsupportedGraph(f"map parameter '{p}' is not a clamped tile of '{b.name}'")
            used.add(b.name)
            b, e = tb, te
        flat[p] = (b, e)
        order.append(p)
    if set(tiles) - used:
        raise UnsupportedGraph("strided map without a matching inner tile map")
    params = set(flat)
    for p, (b, e) in flat.items():
        if (X.free_symbols(b) | X.free_symbols(e)) & (params | set(tiles)):
            raise UnsupportedGraph(f"map range of '{p}' depends on another map parameter")
    return Nest(entries, flat, order, body, local, bind)


def _dynamic_connectors(entry: Node) -> set:
    return {c for c in entry.doc.get("ins", []) if not c.startswith("IN_")}


def _is_local_storage(state: State, node: Node, outer: Node, inner: Node, local: dict) -> bool:
    """Access node of a transient filled by a region copy from ``outer`` and
    read by ``inner`` (LocalStorage, library.py:679-722)."""
    if node.kind != "access":
        return False
    ins = state.in_edges(node.id)
    outs = state.out_edges(node.id)
    if len(ins) != 1 or ins[0].src != outer.id or not outs or any(o.dst != inner.id for o in outs):
        return False
    m = ins[0].memlet
    if m.is_empty or m.reindex is None or m.data == node.data:
        return False
    local[node.data] = (m.data, tuple(r.begin for r in m.subset))
    return True


def resolve_read(state: State, edge, nest: Nest, tile_params: set) -> tuple:
    """``(container, [Affine])`` of a tasklet input after looking through
    LocalStorage transients; indices are affine over the flat parameters."""
    m = edge.memlet
    if m.is_empty:
        raise UnsupportedGraph("empty memlet into a tasklet input")
    data = m.data
    idx = []
    sub = {k: X.Sym(v) for k, v in nest.bind.items()}
    for r in m.subset:
        if not r.is_point:
            raise UnsupportedGraph(f"tasklet input '{edge.dst_conn}' reads a region")
        idx.append(X.substitute(r.begin, sub))
    if data in nest.local:
        orig, origin = nest.local[data]
        idx = [X.Bin("+", a, o) for a, o in zip(idx, origin)]
        data = orig
    aff = []
    for e in idx:
        a = X.affine(e)
        if a is None:
            aff.append(e)  # non-affine (e.g. t % 2): caller inspects
            continue
        if set(a.terms) & tile_params:
            raise UnsupportedGraph(f"index {e} still depends on a tile parameter")
        aff.append(a)
    return data, aff


def _bound(nest: Nest, e: X.Expr) -> X.Expr:
    """An innermost-scope expression in the nest's unique parameter names."""
    return X.substitute(e, {k: X.Sym(v) for k, v in nest.bind.items()})


def _tile_params(nest: Nest) -> set:
    out = set()
    for lvl, e in enumerate(nest.entries):
        out |= {f"{p}#{lvl}" for p in e.params}
    return out - set(nest.flat)


def _covers_full(nest: Nest, params: list, dims: tuple, offset: int = 0) -> bool:
    """flat ranges of ``params`` are [offset : dim-1-offset] of ``dims``."""
    for p, d in zip(params, dims):
        b, e = nest.flat[p]
        if not X.same_value(b, X.Num(offset)):
            return False
        if not X.same_value(e, X.Bin("-", d, X.Num(1 + offset))):
            return False
    return True


def _tasklets(state: State, ids: list) -> list:
    return [state.nodes[i] for i in ids if state.nodes[i].kind == "tasklet"]


def _single_stmt(t: Node) -> ast.stmt:
    body = t.code_ast.body
    if len(body) != 1:
        raise UnsupportedGraph(f"tasklet '{t.name}' has {len(body)} statements")
    return body[0]


def _const(n: ast.AST) -> Optional[float]:
    if isinstance(n, ast.Constant) and isinstance(n.value, (int, float)) and not isinstance(n.value, bool):
        return n.value
    if isinstance(n, ast.UnaryOp) and isinstance(n.op, ast.USub):
        v = _const(n.operand)
        return -v if v is not None else None
    return None


def _exit_write(state: State, t: Node, conn: str) -> list:
    """Final (access node, memlet) targets of tasklet output ``conn``,
    traced through scope exits (codegen.py:261-277 resolve_targets)."""
    out = []
    for e in state.out_edges(t.id):
        if e.src_conn != conn:
            continue
        inner_memlet = e.memlet
        frontier = [e]
        while frontier:
            cur = frontier.pop()
            dst = state.nodes[cur.dst]
            if dst.kind == "access":
                out.append((dst, inner_memlet))
            elif dst.kind in ("map_exit", "consume_exit"):
                oc = "OUT_" + (cur.dst_conn or "")[3:]
                frontier.extend(x for x in state.out_edges(dst.id) if x.src_conn == oc)
            else:
                out.append((dst, inner_memlet))
    return out


def _base(g: Graph, motif: str) -> Plan:
    return Plan(motif, g.name, g.pointer_args(), list(g.symbols), {},
                dims={n: d.dims for n, d in g.data.items()})


def _compute_states(g: Graph) -> list:
    return [s for s in g.states if s.nodes]


def _walk(g: Graph, start: str, until: Optional[str] = None, entry_assign: tuple = ()) -> list:
    """States the interpreter visits from ``start`` (interpreter.py:689-709)
    when control flow is straight-line: every transition taken is the
    first out-transition of its state, unconditional, and assigns nothing
    -- except the one into ``until``, which may carry ``entry_assign``.
    Anything else (a condition, an assignment, a cycle) could run a state
    zero or several times, so the motif kernel, which runs it once, does
    not apply and the graph goes to the generic lowering."""
    seq: list = []
    cur: Optional[str] = start
    while cur is not None and cur != until:
        if cur in seq:
            raise UnsupportedGraph(f"control flow revisits state '{cur}'")
        seq.append(cur)
        outs = g.out_transitions(cur)
        if not outs:
            cur = None
            break
        t = outs[0]
        if t.condition != X.Num(1):
            raise UnsupportedGraph(f"conditional transition out of state '{cur}'")
        assigns = [(k, v) for k, v in t.assignments]
        if assigns and not (t.dst == until and len(assigns) == 1 and assigns[0][0] == entry_assign[0]
                            and X.same_value(assigns[0][1], entry_assign[1])):
            raise UnsupportedGraph(f"transition out of state '{cur}' assigns symbols")
        cur = t.dst
    if until is not None and cur != until:
        raise UnsupportedGraph(f"state '{until}' is not reached by straight-line control flow")
    return seq


def _runs_once(g: Graph, names: list) -> None:
    """The dataflow states ``names`` run exactly once, in this order, and
    nothing else with dataflow runs."""
    seq = _walk(g, g.start_state)
    got = [s for s in seq if g.state(s).nodes]
    if got != names:
        raise UnsupportedGraph(f"dataflow states run as {got}, not once each as {names}")


# ----------------------------------------------------------------- histogram

def match_histogram(g: Graph) -> Plan:
    states = _compute_states(g)
    if len(states) != 1:
        raise UnsupportedGraph("histogram: expects one dataflow state")
    st = states[0]
    _runs_once(g, [st.name])
    parent = st.scope_parent()
    tops = _top_maps(st, parent)
    if len(tops) != 1:
        raise UnsupportedGraph("histogram: expects one top-level map")
    nest = map_nest(st, tops[0], parent)
    tp = _tile_params(nest)
    tks = _tasklets(st, nest.body)
    bump = [t for t in tks if isinstance(_single_stmt(t), ast.Assign)
            and isinstance(_single_stmt(t).targets[0], ast.Subscript)]
    if len(bump) != 1:
        raise UnsupportedGraph("histogram: no subscript-write tasklet")
    bump = bump[0]
    s = _single_stmt(bump)
    tgt = s.targets[0]
    if not (isinstance(tgt.value, ast.Name) and isinstance(tgt.slice, ast.Name) and _const(s.value) == 1):
        raise UnsupportedGraph("histogram: bump tasklet is not 'h[k] = 1'")
    out_conn, key_conn = tgt.value.id, tgt.slice.id
    writes = _exit_write(st, bump, out_conn)
    if len(writes) != 1 or writes[0][1].wcr != "sum":
        raise UnsupportedGraph("histogram: subscript write is not WCR-sum")
    hist = writes[0][0].data
    hd = g.data[hist]
    if len(hd.dims) != 1 or hd.basetype != "int64":
        raise UnsupportedGraph("histogram: target must be a rank-1 int64 container")
    key_edge = [e for e in st.in_edges(bump.id) if e.dst_conn == key_conn]
    if len(key_edge) != 1:
        raise UnsupportedGraph("histogram: key input missing")
    ke = key_edge[0]
    src = st.nodes[ke.src]
    plan = _base(g, "histogram")
    binner = None
    if src.kind == "access" and g.data[src.data].transient:
        # two-tasklet form: binner -> bin scalar -> bump
        feeders = [e for e in st.in_edges(src.id)]
        if len(feeders) != 1 or st.nodes[feeders[0].src].kind != "tasklet":
            raise UnsupportedGraph("histogram: bin scalar not written by a tasklet")
        binner = st.nodes[feeders[0].src]
        if g.data[src.data].basetype != "int64":
            raise UnsupportedGraph("histogram: bin scalar must be int64 (floor cast)")
        bs = _single_stmt(binner)
        if not (isinstance(bs, ast.Assign) and isinstance(bs.targets[0], ast.Name)
                and bs.targets[0].id == feeders[0].src_conn):
            raise UnsupportedGraph("histogram: binner must assign its output")
        v = bs.value
        # bi = v * S // D   (or S * v // D)
        if not (isinstance(v, ast.BinOp) and isinstance(v.op, ast.FloorDiv) and _const(v.right) is not None
                and isinstance(v.left, ast.BinOp) and isinstance(v.left.op, ast.Mult)):
            raise UnsupportedGraph("histogram: binner is not 'bi = v * S // D'")
        mul = v.left
        if isinstance(mul.left, ast.Name) and _const(mul.right) is not None:
            vin, scale = mul.left.id, _const(mul.right)
        elif isinstance(mul.right, ast.Name) and _const(mul.left) is not None:
            vin, scale = mul.right.id, _const(mul.left)
        else:
            raise UnsupportedGraph("histogram: binner is not 'bi = v * S // D'")
        div = _const(v.right)
        if div == 0:
            raise UnsupportedGraph("histogram: zero divisor")
        ie = [e for e in st.in_edges(binner.id) if e.dst_conn == vin]
        if len(ie) != 1:
            raise UnsupportedGraph("histogram: binner input missing")
        img, idx = resolve_read(st, ie[0], nest, tp)
        plan.params.update(mode="scaled", scale=float(scale), div=float(div))
        if g.data[img].basetype != "float64":
            raise UnsupportedGraph("histogram: scaled binning needs a float64 image")
    else:
        img, idx = resolve_read(st, ke, nest, tp)
        if g.data[img].basetype != "int64":
            raise UnsupportedGraph("histogram: direct subscript needs an int64 image")
        plan.motif = "histogram_int"
        plan.params.update(mode="identity")
    if any(t is not bump and t is not binner for t in tks):
        raise UnsupportedGraph("histogram: map body has tasklets besides the binner and the bump")
    others = [n for i in nest.body for n in [st.nodes[i]] if n.kind not in ("tasklet", "access")]
    if others:
        raise UnsupportedGraph("histogram: map body has nodes besides tasklets and the bin scalar")
    imd = g.data[img]
    if len(idx) != len(imd.dims) or len(nest.order) != len(idx):
        raise UnsupportedGraph("histogram: image rank does not match the map")
    for a, p in zip(idx, nest.order):
        if not isinstance(a, X.Affine) or a.only(p) != 0:
            raise UnsupportedGraph("histogram: image must be read at the map point")
    if not _covers_full(nest, nest.order, imd.dims):
        raise UnsupportedGraph("histogram: map does not cover the image")
    plan.roles.update(img=img, hist=hist)
    plan.params["bins"] = hd.dims[0]
    plan.main_state, plan.main_map = st.name, tops[0].id
    return plan


# --------------------------------------------------------------------- query

def match_query(g: Graph) -> Plan:
    states = _compute_states(g)
    if len(states) != 1:
        raise UnsupportedGraph("query: expects one dataflow state")
    st = states[0]
    _runs_once(g, [st.name])
    parent = st.scope_parent()
    tops = _top_maps(st, parent)
    if len(tops) != 1:
        raise UnsupportedGraph("query: expects one top-level map")
    nest = map_nest(st, tops[0], parent)
    tp = _tile_params(nest)
    tks = _tasklets(st, nest.body)
    if len(tks) != 1 or len(nest.order) != 1:
        raise UnsupportedGraph("query: expects one tasklet under a 1-D map")
    t = tks[0]
    s = _single_stmt(t)
    if not (isinstance(s, ast.If) and not s.orelse and isinstance(s.test, ast.Compare)
            and len(s.test.ops) == 1 and type(s.test.ops[0]) in CMP_OPS):
        raise UnsupportedGraph("query: predicate tasklet is not 'if v OP limit: ...'")
    a, b = s.test.left, s.test.comparators[0]
    op = CMP_OPS[type(s.test.ops[0])]
    if not (isinstance(a, ast.Name) and isinstance(b, ast.Name)):
        raise UnsupportedGraph("query: predicate must compare two connectors")
    ins = {e.dst_conn: e for e in st.in_edges(t.id) if not e.memlet.is_empty}
    assigns = {}
    for stmt in s.body:
        if not (isinstance(stmt, ast.Assign) and isinstance(stmt.targets[0], ast.Name)):
            raise UnsupportedGraph("query: predicate body must be plain assignments")
        assigns[stmt.targets[0].id] = stmt.value
    push = cnt = None
    for conn, val in assigns.items():
        for acc, m in _exit_write(st, t, conn):
            d = g.data[acc.data]
            if d.kind == "stream" and isinstance(val, ast.Name):
                push = (conn, val.id, acc)
            elif m.wcr == "sum" and _const(val) == 1 and d.basetype == "int64":
                cnt = acc.data
    if push is None or cnt is None:
        raise UnsupportedGraph("query: needs a stream push of the value and a WCR-sum count")
    vconn = push[1]
    if vconn == a.id:
        lconn = b.id
    elif vconn == b.id:
        lconn, op = a.id, MIRROR[op]
    else:
        raise UnsupportedGraph("query: pushed value is not the compared value")
    col, cidx = resolve_read(st, ins[vconn], nest, tp)
    thr, tidx = resolve_read(st, ins[lconn], nest, tp)
    p = nest.order[0]
    if not (isinstance(cidx[0], X.Affine) and cidx[0].only(p) == 0):
        raise UnsupportedGraph("query: column must be read at the map point")
    if not (len(tidx) == 1 and isinstance(tidx[0], X.Affine) and tidx[0].is_const() and tidx[0].const == 0):
        raise UnsupportedGraph("query: limit must be a scalar read")
    if not _covers_full(nest, nest.order, g.data[col].dims):
        raise UnsupportedGraph("query: map does not cover the column")
    stream = push[2]
    drains = [st.nodes[e.dst] for e in st.out_edges(stream.id)
              if st.nodes[e.dst].kind == "access" and g.data[st.nodes[e.dst].data].kind == "array"]
    if len(drains) != 1:
        raise UnsupportedGraph("query: stream must drain into one array")
    out = drains[0].data
    for c in (col, thr, out):
        if g.data[c].basetype != "float64":
            raise UnsupportedGraph("query: column/threshold/output must be float64")
    plan = _base(g, "query")
    plan.roles.update(col=col, thr=thr, out_vals=out, count=cnt)
    plan.params.update(op=op)
    plan.main_state, plan.main_map = st.name, tops[0].id
    return plan


# ---------------------------------------------------------------------- spmv

def match_spmv(g: Graph) -> Plan:
    states = _compute_states(g)
    if len(states) != 1:
        raise UnsupportedGraph("spmv: expects one dataflow state")
    st = states[0]
    _runs_once(g, [st.name])
    parent = st.scope_parent()
    tops = _top_maps(st, parent)
    if len(tops) != 1:
        raise UnsupportedGraph("spmv: expects one top-level map")
    outer = map_nest(st, tops[0], parent)
    inner = [st.nodes[k] for k in outer.body if st.nodes[k].kind == "map_entry"]
    if len(inner) != 1 or len(outer.order) != 1:
        raise UnsupportedGraph("spmv: expects a row map around a data-dependent inner map")
    ime = inner[0]
    dyn = _dynamic_connectors(ime)
    if len(ime.params) != 1 or len(dyn) != 2:
        raise UnsupportedGraph("spmv: inner map needs two data-dependent range connectors")
    i, j = outer.order[0], ime.params[0]
    rng = ime.ranges[0]
    tp = _tile_params(outer)
    conn_src = {}
    for e in st.in_edges(ime.id):
        if e.dst_conn in dyn:
            conn_src[e.dst_conn] = resolve_read(st, e, outer, tp)
    # range  b : e - 1  with b <- rowptr[i], e <- rowptr[i + 1]
    if not (isinstance(rng.begin, X.Sym) and rng.begin.name in conn_src):
        raise UnsupportedGraph("spmv: inner range must start at a range connector")
    fe = X.affine(rng.end)
    bname = rng.begin.name
    ename = [c for c in dyn if c != bname][0]
    if fe is None or fe.only(ename) != -1:
        raise UnsupportedGraph("spmv: inner range must end at connector - 1")
    rp_b, ib = conn_src[bname]
    rp_e, ie = conn_src[ename]
    if rp_b != rp_e or ib[0].only(i) != 0 or ie[0].only(i) != 1:
        raise UnsupportedGraph("spmv: range connectors must be rowptr[i], rowptr[i+1]")
    rowptr = rp_b
    iparent = {k: v for k, v in parent.items()}
    body = [k for k in _children(iparent, ime.id) if st.nodes[k].kind != "map_exit"]
    tks = _tasklets(st, body)
    deref = [t for t in tks if isinstance(_single_stmt(t), ast.Assign)
             and isinstance(_single_stmt(t).value, ast.Subscript)]
    mac = [t for t in tks if t not in deref]
    if len(deref) != 1 or len(mac) != 1:
        raise UnsupportedGraph("spmv: expects an indirection tasklet and a multiply tasklet")
    d, m = deref[0], mac[0]
    ds = _single_stmt(d)
    if not (isinstance(ds.value.value, ast.Name) and isinstance(ds.value.slice, ast.Name)):
        raise UnsupportedGraph("spmv: indirection is not 'out = table[index]'")
    table_conn, index_conn = ds.value.value.id, ds.value.slice.id
    nest_in = type(outer)(outer.entries + [ime], dict(outer.flat, **{j: (rng.begin, rng.end)}),
                          outer.order + [j], body, outer.local)
    din = {e.dst_conn: e for e in st.in_edges(d.id)}
    colc, cidx = resolve_read(st, din[index_conn], nest_in, tp)
    te = din[table_conn].memlet
    xvec = te.data
    if cidx[0].only(j) != 0 or len(te.subset) != 1 or te.subset[0].is_point:
        raise UnsupportedGraph("spmv: indirection must read index[j] into a whole vector")
    ms = _single_stmt(m)
    if not (isinstance(ms, ast.Assign) and isinstance(ms.value, ast.BinOp) and isinstance(ms.value.op, ast.Mult)
            and isinstance(ms.value.left, ast.Name) and isinstance(ms.value.right, ast.Name)):
        raise UnsupportedGraph("spmv: multiply tasklet is not 'out = a * b'")
    min_ = {e.dst_conn: e for e in st.in_edges(m.id)}
    val = None
    for c in (ms.value.left.id, ms.value.right.id):
        e = min_[c]
        srcn = st.nodes[e.src]
        if srcn.kind == "access" and g.data[srcn.data].transient:
            feed = st.in_edges(srcn.id)
            if len(feed) != 1 or feed[0].src != d.id:
                raise UnsupportedGraph("spmv: gathered scalar must come from the indirection")
        else:
            val, vidx = resolve_read(st, e, nest_in, tp)
            if vidx[0].only(j) != 0:
                raise UnsupportedGraph("spmv: values must be read at j")
    if val is None:
        raise UnsupportedGraph("spmv: no matrix values input")
    writes = _exit_write(st, m, ms.targets[0].id)
    if len(writes) != 1 or writes[0][1].wcr != "sum":
        raise UnsupportedGraph("spmv: product must accumulate with WCR sum")
    b = writes[0][0].data
    bidx = [X.affine(_bound(outer, r.begin)) for r in writes[0][1].subset]
    if len(bidx) != 1 or bidx[0] is None or bidx[0].only(i) != 0:
        raise UnsupportedGraph("spmv: accumulation target must be b[i]")
    if not _covers_full(outer, [i], g.data[b].dims):
        raise UnsupportedGraph("spmv: row map does not cover b")
    for c, bt in ((rowptr, "int64"), (colc, "int64"), (val, "float64"), (xvec, "float64"), (b, "float64")):
        if g.data[c].basetype != bt:
            raise UnsupportedGraph(f"spmv: '{c}' must be {bt}")
    plan = _base(g, "spmv")
    plan.roles.update(rowptr=rowptr, col=colc, val=val, x=xvec, b=b)
    plan.main_state, plan.main_map = st.name, tops[0].id
    return plan


# ------------------------------------------------------------------ jacobi2d

@dataclass
class Loop:
    guard: str
    body: str
    var: str
    count: X.Expr


def detect_loop(g: Graph) -> Optional[Loop]:
    """Guard loop ``for (v = 0; v < count; v = v + 1)`` (loops.py:31-61 restated)."""
    for guard in g.states:
        if guard.nodes:
            continue
        outs = g.out_transitions(guard.name)
        if not outs or outs[0].condition == X.Num(1):
            continue
        enter = outs[0]
        body = g.state(enter.dst)
        if body is None or body.name == guard.name:
            continue
        back = g.out_transitions(body.name)
        if len(back) != 1 or back[0].dst != guard.name or len(back[0].assignments) != 1:
            continue
        var, upd = back[0].assignments[0]
        fu = X.affine(upd)
        if fu is None or fu.only(var) != 1:
            continue
        entries = [t for t in g.in_transitions(guard.name) if t.src != body.name]
        inits = [dict(t.assignments).get(var) for t in entries]
        if not entries or any(v is None or not X.same_value(v, X.Num(0)) for v in inits):
            continue
        c = enter.condition
        if isinstance(c, X.Cmp) and isinstance(c.left, X.Sym) and c.left.name == var:
            if c.op == "<":
                count = c.right
            elif c.op == "<=":
                count = X.Bin("+", c.right, X.Num(1))
            else:
                continue
            if var in X.free_symbols(count):
                continue
            return Loop(guard.name, body.name, var, count)
    return None


def _loop_runs_once(g: Graph, loop: Loop) -> None:
    """The guard loop is entered once from straight-line code (``v = 0`` on
    the entering edge), its body is reached only from the guard, and the
    exit leads straight to the end -- so the device-side T loop is the
    whole program (interpreter.py:689-709)."""
    _walk(g, g.start_state, until=loop.guard, entry_assign=(loop.var, X.Num(0)))
    ins = g.in_transitions(loop.guard)
    if len(ins) != 2 or len(g.in_transitions(loop.body)) != 1:
        raise UnsupportedGraph("jacobi2d: guard loop is entered from more than one place")
    outs = g.out_transitions(loop.guard)
    if len(outs) > 2:
        raise UnsupportedGraph("jacobi2d: guard state has more than two exits")
    if len(outs) == 2:
        t = outs[1]
        if t.condition != X.Num(1) or t.assignments:
            raise UnsupportedGraph("jacobi2d: guard exit is conditional or assigns symbols")
        after = _walk(g, t.dst)
        if loop.guard in after or any(g.state(s).nodes for s in after):
            raise UnsupportedGraph("jacobi2d: dataflow or a loop after the time loop")


def _sum_chain(n: ast.AST) -> Optional[list]:
    """Names of a left-leaning ``((a + b) + c) + ...`` chain, in order."""
    if isinstance(n, ast.Name):
        return [n.id]
    if isinstance(n, ast.BinOp) and isinstance(n.op, ast.Add) and isinstance(n.right, ast.Name):
        left = _sum_chain(n.left)
        return left + [n.right.id] if left is not None else None
    return None


def match_jacobi(g: Graph) -> Plan:
    loop = detect_loop(g)
    if loop is None:
        raise UnsupportedGraph("jacobi2d: no guard loop")
    others = [s for s in g.states if s.name != loop.body and s.nodes]
    if others:
        raise UnsupportedGraph("jacobi2d: dataflow outside the loop body")
    _loop_runs_once(g, loop)
    st = g.state(loop.body)
    parent = st.scope_parent()
    tops = _top_maps(st, parent)
    if len(tops) != 1:
        raise UnsupportedGraph("jacobi2d: expects one top-level map in the body")
    nest = map_nest(st, tops[0], parent)
    tp = _tile_params(nest)
    tks = _tasklets(st, nest.body)
    if len(tks) != 1 or len(nest.order) != 2:
        raise UnsupportedGraph("jacobi2d: expects one tasklet under a 2-D map")
    t = tks[0]
    s = _single_stmt(t)
    if not (isinstance(s, ast.Assign) and isinstance(s.targets[0], ast.Name)
            and isinstance(s.value, ast.BinOp) and isinstance(s.value.op, ast.Mult)):
        raise UnsupportedGraph("jacobi2d: tasklet is not 'o = coef * (sum)'")
    if _const(s.value.left) is not None:
        coef, chain = _const(s.value.left), _sum_chain(s.value.right)
    else:
        coef, chain = _const(s.value.right), _sum_chain(s.value.left)
    if coef is None or chain is None or not 1 <= len(chain) <= 9:
        raise UnsupportedGraph("jacobi2d: tasklet is not 'o = coef * (t0 + t1 + ...)'")
    pi, pj = nest.order
    tvar = X.Sym(loop.var)
    cur_plane = X.Bin("%", tvar, X.Num(2))
    nxt_plane = X.Bin("%", X.Bin("+", tvar, X.Num(1)), X.Num(2))
    ins = {e.dst_conn: e for e in st.in_edges(t.id)}
    arr = None
    terms = []
    for name in chain:
        if name not in ins:
            raise UnsupportedGraph(f"jacobi2d: '{name}' is not an input connector")
        data, idx = resolve_read(st, ins[name], nest, tp)
        if len(idx) != 3 or idx[0] != cur_plane:
            raise UnsupportedGraph("jacobi2d: reads must be A[t % 2, i + di, j + dj]")
        di, dj = idx[1].only(pi) if isinstance(idx[1], X.Affine) else None, \
            idx[2].only(pj) if isinstance(idx[2], X.Affine) else None
        if di is None or dj is None or abs(di) > 1 or abs(dj) > 1:
            raise UnsupportedGraph("jacobi2d: neighbour offsets must be within 1")
        if arr not in (None, data):
            raise UnsupportedGraph("jacobi2d: all reads must come from one container")
        arr = data
        terms.append((int(di), int(dj)))
    writes = _exit_write(st, t, s.targets[0].id)
    if len(writes) != 1 or writes[0][1].wcr is not None or writes[0][0].data != arr:
        raise UnsupportedGraph("jacobi2d: result must be written (no WCR) into the same container")
    w = [_bound(nest, r.begin) for r in writes[0][1].subset]
    if not (len(w) == 3 and w[0] == nxt_plane
            and X.affine(w[1]) is not None and X.affine(w[1]).only(pi) == 0
            and X.affine(w[2]) is not None and X.affine(w[2]).only(pj) == 0):
        raise UnsupportedGraph("jacobi2d: write must be A[(t + 1) % 2, i, j]")
    d = g.data[arr].dims
    if len(d) != 3 or not X.same_value(d[0], X.Num(2)) or not X.same_value(d[1], d[2]):
        raise UnsupportedGraph("jacobi2d: container must be [2, N, N]")
    if not _covers_full(nest, [pi, pj], d[1:], offset=1):
        raise UnsupportedGraph("jacobi2d: map must cover the interior [1:N-2]^2")
    if g.data[arr].basetype != "float64":
        raise UnsupportedGraph("jacobi2d: container must be float64")
    plan = _base(g, "jacobi2d")
    plan.roles.update(A=arr)
    plan.params.update(coef=float(coef), terms=terms, steps=loop.count, N=d[1])
    plan.main_state, plan.main_map = st.name, tops[0].id
    return plan


# -------------------------------------------------------------------- matmul

def _mm_core(g: Graph, st: State, nest: Nest, t: Node) -> tuple:
    s = _single_stmt(t)
    if not (isinstance(s, ast.Assign) and isinstance(s.targets[0], ast.Name) and isinstance(s.value, ast.BinOp)
            and isinstance(s.value.op, ast.Mult) and isinstance(s.value.left, ast.Name)
            and isinstance(s.value.right, ast.Name)):
        raise UnsupportedGraph("matmul: tasklet is not 'o = a * b'")
    tp = _tile_params(nest)
    ins = {e.dst_conn: e for e in st.in_edges(t.id)}
    reads = [resolve_read(st, ins[c], nest, tp) for c in (s.value.left.id, s.value.right.id)]
    return s, reads


def _mm_roles(nest: Nest, reads: list, out_idx: list) -> tuple:
    """Identify (A, B, i, j, k) from A[i, k], B[k, j], out[i, j]."""
    def var(a):
        return next(iter(a.terms)) if isinstance(a, X.Affine) and len(a.terms) == 1 and a.const == 0 \
            and list(a.terms.values()) == [1] else None
    oi, oj = (var(a) for a in out_idx)
    if oi is None or oj is None or oi == oj:
        raise UnsupportedGraph("matmul: output must be C[i, j]")
    for (ra, ia), (rb, ib) in (reads, reads[::-1]):
        a0, a1 = (var(x) for x in ia)
        b0, b1 = (var(x) for x in ib)
        if a0 == oi and b1 == oj and a1 is not None and a1 == b0 and a1 not in (oi, oj):
            return ra, rb, oi, oj, a1
    raise UnsupportedGraph("matmul: inputs are not A[i, k] and B[k, j]")


def match_matmul(g: Graph) -> Plan:
    states = _compute_states(g)
    plan = _base(g, "matmul")
    if len(states) == 2:
        # MapReduceFusion form: init state (C = identity) then the fused map
        init, mult = None, None
        for st in states:
            parent = st.scope_parent()
            tops = _top_maps(st, parent)
            if len(tops) != 1:
                raise UnsupportedGraph("matmul: expects one map per state")
            nest = map_nest(st, tops[0], parent)
            tks = _tasklets(st, nest.body)
            if len(tks) != 1:
                raise UnsupportedGraph("matmul: expects one tasklet per state")
            s = _single_stmt(tks[0])
            if isinstance(s, ast.Assign) and _const(s.value) is not None:
                init = (st, nest, tks[0], s, tops[0])
            else:
                mult = (st, nest, tks[0], tops[0])
        if init is None or mult is None:
            raise UnsupportedGraph("matmul: needs an init state and a multiply state")
        ist, inest, itk, istmt, _ = init
        if _const(istmt.value) != 0:
            raise UnsupportedGraph("matmul: init must write the sum identity 0")
        _runs_once(g, [ist.name, mult[0].name])
        st, nest, t, top = mult
        s, reads = _mm_core(g, st, nest, t)
        writes = _exit_write(st, t, s.targets[0].id)
        if len(writes) != 1 or writes[0][1].wcr != "sum":
            raise UnsupportedGraph("matmul: product must accumulate with WCR sum")
        C = writes[0][0].data
        out_idx = [X.affine(_bound(nest, r.begin)) for r in writes[0][1].subset]
        iw = _exit_write(ist, itk, istmt.targets[0].id)
        if len(iw) != 1 or iw[0][0].data != C or not _covers_full(inest, inest.order, g.data[C].dims):
            raise UnsupportedGraph("matmul: init must cover C")
    elif len(states) == 1:
        # raw form: map -> tmp[i, j, k] -> Reduce(axes=[2], sum) -> C
        st = states[0]
        _runs_once(g, [st.name])
        parent = st.scope_parent()
        tops = _top_maps(st, parent)
        if len(tops) != 1:
            raise UnsupportedGraph("matmul: expects one top-level map")
        top = tops[0]
        nest = map_nest(st, top, parent)
        tks = _tasklets(st, nest.body)
        if len(tks) != 1:
            raise UnsupportedGraph("matmul: expects one tasklet")
        t = tks[0]
        s, reads = _mm_core(g, st, nest, t)
        writes = _exit_write(st, t, s.targets[0].id)
        if len(writes) != 1 or writes[0][1].wcr is not None:
            raise UnsupportedGraph("matmul: raw product must be materialised")
        tmp = writes[0][0]
        red = [st.nodes[e.dst] for e in st.out_edges(tmp.id)]
        if len(red) != 1 or red[0].kind != "reduce" or (red[0].doc.get("wcr") or {}).get("kind") != "sum":
            raise UnsupportedGraph("matmul: product must feed a sum Reduce")
        tidx = [X.affine(_bound(nest, r.begin)) for r in writes[0][1].subset]
        axes = red[0].doc["axes"]
        if len(tidx) != 3 or list(axes) != [2]:
            raise UnsupportedGraph("matmul: Reduce must contract the last axis of tmp[i, j, k]")
        outs = [st.nodes[e.dst] for e in st.out_edges(red[0].id)]
        if len(outs) != 1 or outs[0].kind != "access":
            raise UnsupportedGraph("matmul: Reduce must write one container")
        C = outs[0].data
        out_idx = tidx[:2]
        k_from_tmp = tidx[2]
        if not (isinstance(k_from_tmp, X.Affine) and len(k_from_tmp.terms) == 1):
            raise UnsupportedGraph("matmul: tmp must be indexed [i, j, k]")
    else:
        raise UnsupportedGraph("matmul: unexpected state structure")
    A, B, i, j, k = _mm_roles(nest, reads, out_idx)
    da, db, dc = g.data[A].dims, g.data[B].dims, g.data[C].dims
    if not (len(da) == len(db) == len(dc) == 2):
        raise UnsupportedGraph("matmul: operands must be rank 2")
    if not (_covers_full(nest, [i, k], da) and _covers_full(nest, [k, j], db) and _covers_full(nest, [i, j], dc)):
        raise UnsupportedGraph("matmul: map does not cover the operands")
    for c in (A, B, C):
        if g.data[c].basetype != "float64":
            raise UnsupportedGraph("matmul: operands must be float64")
    plan.roles.update(A=A, B=B, C=C)
    plan.main_state, plan.main_map = st.name, top.id
    return plan


MATCHERS = (match_histogram, match_query, match_spmv, match_jacobi, match_matmul)


def classify(g: Graph) -> Plan:
    reasons = []
    for m in MATCHERS:
        try:
            return m(g)
        except UnsupportedGraph as exc:
            reasons.append(str(exc))
        except (KeyError, IndexError, AttributeError, TypeError) as exc:
            reasons.append(f"{m.__name__}: {type(exc).__name__}: {exc}")
    raise UnsupportedGraph(f"no sm_100a motif matches SDFG '{g.name}':\n  " + "\n  ".join(reasons))
