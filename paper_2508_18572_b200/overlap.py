"""Layer-wise overlap model for consumers of the per-layer completion events.

The executor waits until layer l's KV is loaded before running layer l (§4.1), so
prefill of layer l overlaps the loading of later layers ("layer-wise overlapping approach",
PAPER.md:281 §4.2.1).  With per-layer load times t_load[l] issued back to back and
per-layer compute t_comp[l], the finish times follow the recurrence of SPEC.md:376 (engine
prefill_wall_time):

    load_finish[l] = load_finish[l-1] + t_load[l]
    comp_finish[l] = max(comp_finish[l-1], load_finish[l]) + t_comp[l]
    wall = comp_finish[L-1],  stall = wall - sum(t_comp)

Used to check measured overlap against the model (tools/overlap.py, tests/test_gpu_overlap.py) and
pinned on CPU against SPEC.md's hand-evaluated examples (tests/golden/pipeline_recurrence.json).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def pipeline_recurrence(t_load: Sequence[float], t_comp: Sequence[float],
                        load_finish: Sequence[float] = None) -> Tuple[List[float], float, float]:
    """Return (comp_finish per layer, wall, stall).  ``load_finish`` (absolute completion times of
    the layer loads, e.g. measured from the per-layer events) overrides the cumulative sum."""
    if len(t_load) != len(t_comp):
        raise ValueError("t_load and t_comp must have one entry per layer")
    if load_finish is None:
        load_finish, acc = [], 0.0
        for t in t_load:
            acc += t
            load_finish.append(acc)
    comp, prev = [], 0.0
    for lf, tc in zip(load_finish, t_comp):
        prev = max(prev, lf) + tc
        comp.append(prev)
    wall = comp[-1] if comp else 0.0
    return comp, wall, wall - sum(t_comp)
