"""Seeded request traces for the control plane (NEXT-4).  No scheduling arithmetic lives here.

The paper's workloads are long shared documents with several questions each (LooGLE: avg. 21,613
input tokens; NarrativeQA: 54,797; Table 1) and multi-round conversations whose
rounds extend each other ("preserve dependencies across conversation rounds"). The
order in which requests on the same document arrive is the "cache distance" knob of §5.3.2
(min distance: questions on one document back to back; max: round-robin over documents).

Token ids are drawn uniformly from [0, vocab); documents are independent draws, so two documents
share no prefix beyond chance.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

__all__ = ["shared_context_trace", "conversation_trace", "random_prefix_family"]


def shared_context_trace(rng: np.random.Generator, docs: int, questions: int, doc_len: int,
                         q_len: Tuple[int, int], vocab: int = 32000, order: str = "min",
                         system_prompt: int = 0, return_docs: bool = False):
    """Requests = [system prompt] + document + question.

    order "min": the questions of a document arrive back to back (minimum cache distance);
    "max": round-robin over documents (maximum distance); "random": shuffled.
    return_docs: also return each document's context (system prompt + document).
    """
    sp = rng.integers(0, vocab, system_prompt).tolist()
    bodies = [rng.integers(0, vocab, doc_len).tolist() for _ in range(docs)]
    reqs = [[sp + bodies[d] + rng.integers(0, vocab, int(rng.integers(q_len[0], q_len[1] + 1))).tolist()
             for _ in range(questions)] for d in range(docs)]
    if order == "min":
        out = [r for d in range(docs) for r in reqs[d]]
    elif order == "max":
        out = [reqs[d][q] for q in range(questions) for d in range(docs)]
    else:
        flat = [r for d in range(docs) for r in reqs[d]]
        out = [flat[i] for i in rng.permutation(len(flat))]
    return (out, [sp + b for b in bodies]) if return_docs else out


def conversation_trace(rng: np.random.Generator, convs: int, rounds: int, first_len: Tuple[int, int],
                       turn_len: Tuple[int, int], answer_len: Tuple[int, int],
                       vocab: int = 32000) -> List[List[List[int]]]:
    """Per conversation, the token list of each round: round j = round j-1 + answer + new turn."""
    out = []
    for _ in range(convs):
        toks = rng.integers(0, vocab, int(rng.integers(first_len[0], first_len[1] + 1))).tolist()
        conv = [list(toks)]
        for _ in range(rounds - 1):
            toks = toks + rng.integers(0, vocab, int(rng.integers(answer_len[0], answer_len[1] + 1))).tolist()
            toks = toks + rng.integers(0, vocab, int(rng.integers(turn_len[0], turn_len[1] + 1))).tolist()
            conv.append(list(toks))
        out.append(conv)
    return out


def random_prefix_family(rng: np.random.Generator, count: int, max_len: int, vocab: int,
                         branch: float = 0.5) -> List[List[int]]:
    """Small sequences that share prefixes often (for brute-force tree tests): each new sequence
    copies a random prefix of an earlier one with probability `branch`, then appends fresh tokens."""
    seqs: List[List[int]] = []
    for _ in range(count):
        n = int(rng.integers(1, max_len + 1))
        if seqs and rng.random() < branch:
            base = seqs[int(rng.integers(0, len(seqs)))]
            cut = int(rng.integers(0, len(base) + 1))
            s = base[:min(cut, n)]
        else:
            s = []
        s = s + rng.integers(0, vocab, max(0, n - len(s))).tolist()
        seqs.append(s[:n])
    return seqs
