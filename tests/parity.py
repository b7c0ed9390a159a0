"""Free-running greedy parity with explicit near-tie reporting (SURVEY.md
§8(c) T4a) -- test infrastructure only.

Reading of "identical greedy ids": the GPU's ids equal the oracle's
(mode iii) free-running.  A mismatch at a step whose oracle top-2 margin
exceeds 2*tol is a hard failure.  A mismatch below that is a near-tie
divergence: it is recorded (printed, collected into NEAR_TIES and listed in
the pytest terminal summary -- never passed silently), the GPU's token must
lie within 2*tol of the oracle's maximum, and the rest of that request keeps
being checked: from the next step on, against the oracle teacher-forced on the
GPU's own tokens (the GPU's later steps consumed its own token), logits
within tol on every step, ids equal to the teacher-forced argmax except at
further near ties (also recorded).
"""
from typing import Callable, List, Optional

import numpy as np

NEAR_TIES: List[tuple] = []


def argmax_first(v):
    m = v.max()
    return int(np.flatnonzero(v == m)[0])


def top2(v):
    s = np.sort(v)
    return float(s[-1] - s[-2])


def compare_free_running(label: str, toks, logits, ora, tol: float,
                         teacher_forced: Optional[Callable[[int, List[int]], List[np.ndarray]]],
                         requests=None, max_near_ties: int = 1, tol_mean: Optional[float] = None,
                         steps: Optional[int] = None):
    """toks[r] / logits[r][t]: GPU ids and fp32 logits of request r (logits
    may cover a subset of requests: those with logits[r] non-empty are
    checked).  ora: oracle Result (tokens, logits, margins) for the same
    requests (same indexing).  teacher_forced(r, gpu_tokens) -> oracle logits
    per step with the decode inputs forced to the GPU's tokens.  Returns
    (max-abs, mean-abs, events)."""
    worst = worst_mean = 0.0
    events = []
    for r in range(len(ora.tokens)):
        if logits is not None and not len(logits[r]):
            continue
        k = len(ora.tokens[r]) if steps is None else min(steps, len(ora.tokens[r]))
        ref, ref_tok, ref_margin = ora.logits[r], ora.tokens[r], ora.margins[r]
        diverged = False
        for t in range(k):
            if logits is not None:
                d = np.abs(np.asarray(logits[r][t], np.float64) - ref[t])
                worst, worst_mean = max(worst, float(d.max())), max(worst_mean, float(d.mean()))
            if toks[r][t] != ref_tok[t]:
                m = ref_margin[t]
                assert m <= 2 * tol, "%s: hard mismatch req %d step %d (oracle margin %.4g > 2 tol)" % (label, r, t, m)
                assert ref[t][toks[r][t]] >= ref[t].max() - 2 * tol, (label, r, t)
                ev = (label, r, t, float(m))
                events.append(ev)
                print("NEAR-TIE %s: request %d step %d, oracle top-2 margin %.3g (gpu %d, oracle %d)"
                      % (label, r, t, m, toks[r][t], ref_tok[t]))
                if teacher_forced is None or t + 1 >= k:
                    break
                if not diverged:
                    # from here on the GPU consumed its own tokens: compare with the
                    # oracle teacher-forced on them
                    diverged = True
                    ref = teacher_forced(r, list(toks[r][:k]))
                    ref_tok = [argmax_first(v) for v in ref]
                    ref_margin = [top2(v) for v in ref]
    NEAR_TIES.extend(events)
    assert worst <= tol, "%s: max |logit diff| %.4g > %.4g" % (label, worst, tol)
    if tol_mean is not None:
        assert worst_mean <= tol_mean, "%s: mean |logit diff| %.4g > %.4g" % (label, worst_mean, tol_mean)
    assert len(events) <= max_near_ties, events
    return worst, worst_mean, events


def decoder_only_tf(W, requests, mode="bf16", accum="fp64"):
    """teacher_forced callback for oracle/transformer.py (decoder-only)."""
    from oracle import transformer as T

    def f(r, forced):
        return T.teacher_forced_logits(W, requests[r], forced, mode, accum=accum)
    return f


def t5_tf(W, requests, mode="bf16"):
    """teacher_forced callback for oracle/t5.py."""
    from oracle import t5 as T5

    def f(r, forced):
        res = T5.greedy_kv(W, [requests[r]], mode, record_logits=True, forced=[forced])
        return res.logits[0]
    return f
