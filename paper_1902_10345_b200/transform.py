"""``GPUTransformMap``: the plug-in rule that hands a Map scope to the B200.

It is a transformation in the reference's own framework (engine.py:81-115):
a one-node pattern on a ``MapEntry`` (like MapTiling, library.py:565-566),
an applicability check, and a rewrite on the copy that
``apply_transformation`` makes (engine.py:178-202).  The rule applies to the
top-level map of the program's compute state when the whole program is a
motif the sm_100a library implements (classify.py); ``apply`` records the
decision -- and the ``precision`` and ``stream_order`` parameters, which are
journaled like any rule parameter (engine.py:188-202) -- in
``DataDesc.storage`` of the motif's containers.  ``stream_order`` "any"
(default) lets concurrent pushes land in any order (a Stream is a concurrent
queue); "fifo" keeps the generated C code's input order.
``storage`` is a free string (ir.py:75) the validator and the interpreter
ignore, so the marked graph stays valid for the reference's interpreter,
which remains the oracle for it (the reference rejects any new map
schedule, validation.py:122-125, and has no GPU transformation, so the
marker cannot be a schedule).

Registration is explicit (``paper_1902_10345_b200.register()``): adding a
15th rule to the reference registry changes ``sorted(registry)``, which one
reference acceptance test pins (test_acceptance.py:144).
"""

from __future__ import annotations

from typing import Any

from .classify import UnsupportedGraph, classify
from .dispatch import PRECISIONS, STORAGE_PREFIX, STREAM_ORDERS, gpu_storage
from .graph import load

RULE_NAME = "GPUTransformMap"


def build_rule(engine, matching, ir):
    """Create the rule class against the given reference modules."""

    class GPUTransformMap(engine.Transformation):
        name = RULE_NAME
        strict = False
        default_params = {"precision": "native", "stream_order": "any"}

        def expressions(self):
            return [matching.Pattern([matching.PatternNode("map", (ir.MapEntry,))])]

        def _plan(self, sdfg):
            try:
                return classify(load(sdfg))
            except (UnsupportedGraph, ValueError, KeyError):
                return None

        def _generic(self, sdfg):
            """A graph outside the motifs the generic lowering accepts: the
            rule matches its first top-level map (state order, node order)."""
            from .lower import LoweringError, lower
            try:
                g = load(sdfg)
                lower(g)
            except (LoweringError, ValueError, KeyError):
                return None
            for st in g.states:
                parent = st.scope_parent()
                for n in st.nodes:
                    if n.kind == "map_entry" and parent[n.id] is None:
                        return g, st.name, n.id
            return None

        def can_be_applied(self, sdfg, state, match, strict=False):
            plan = self._plan(sdfg)
            entry = match.nodes["map"]
            if plan is None:
                gen = self._generic(sdfg)
                if gen is None or gen[1] != state.name or sorted(state.nodes).index(entry) != gen[2]:
                    return False
                return not all((d.storage or "").startswith(STORAGE_PREFIX)
                               for d in sdfg.data.values() if not d.transient)
            if plan.main_state != state.name:
                return False
            # to_json renumbers node ids densely in id order (serialization.py:113-116)
            if sorted(state.nodes).index(entry) != plan.main_map:
                return False
            return not all((sdfg.data[c].storage or "").startswith(STORAGE_PREFIX)
                           for c in plan.roles.values())

        def apply(self, sdfg, state, match, params):
            prec = params.get("precision", "native")
            if prec not in PRECISIONS:
                raise ValueError(f"precision must be one of {PRECISIONS}, not '{prec}'")
            order = params.get("stream_order", "any")
            if order not in STREAM_ORDERS:
                raise ValueError(f"stream_order must be one of {STREAM_ORDERS}, not '{order}'")
            plan = self._plan(sdfg)
            if plan is not None:
                for c in set(plan.roles.values()):
                    sdfg.data[c].storage = gpu_storage(prec, order)
                return
            if self._generic(sdfg) is None:
                raise ValueError("GPUTransformMap: program is neither a B200 motif nor lowerable")
            for name, d in sdfg.data.items():
                if not d.transient:
                    d.storage = gpu_storage(prec, order)

    return GPUTransformMap


def register(rewriting: Any = None):
    """Register GPUTransformMap into the reference registry (engine.register,
    engine.py:110-115).  ``rewriting`` defaults to ``import sdfg.rewriting``."""
    if rewriting is None:
        import importlib
        rewriting = importlib.import_module("sdfg.rewriting")
    pkg = rewriting.__name__.rsplit(".", 1)[0]
    import importlib
    engine = importlib.import_module(rewriting.__name__ + ".engine")
    matching = importlib.import_module(rewriting.__name__ + ".matching")
    ir = importlib.import_module(pkg + ".ir")
    if RULE_NAME in engine.registry:
        return type(engine.registry[RULE_NAME])
    cls = build_rule(engine, matching, ir)
    engine.register(cls)
    return cls


def unregister(rewriting: Any = None) -> None:
    if rewriting is None:
        import importlib
        rewriting = importlib.import_module("sdfg.rewriting")
    import importlib
    engine = importlib.import_module(rewriting.__name__ + ".engine")
    engine.registry.pop(RULE_NAME, None)
