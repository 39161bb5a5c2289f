"""Predictor parity: the reference's `specpipe verify` scenarios that need no
crypto (cli.py:217-238), the classification rules (predictor.py:63-94), and
the incremental recognizer against the from-scratch definition on random
histories."""
from __future__ import annotations

import random

import pytest

from paper_2411_03357_b200.predictor import (
    AmbiguousProfile, ModelProfile, PatternKind, Predictor, PredictorConfig, SwapHistory, TransferClass,
    UnknownBlock, classify, outstanding_groups, predict_batches, predict_next, recognize,
)

MIB = 1 << 20


def test_verify_repetitive():
    """cli.py:217-226 (Fig 4a): history [1,3,4,1] predicts 3."""
    h = SwapHistory()
    for b in (1, 3, 4):
        h.observe_swap_out(b)
    for b in (1, 3, 4, 1):
        h.observe_swap_in([b])
        h.observe_swap_out(b)
    assert [p.block for p in predict_next(h, h.outstanding, current_iv=10, leeway=0, depth=1)] == [3]


def test_verify_lifo_reproduces_reference_defect_c1():
    """cli.py:229-238 expects [2, 1] but the reference predicts [] (period-1
    suffix -> REPETITIVE beats LIFO, cycle entry not outstanding).  Parity
    means reproducing []."""
    h = SwapHistory()
    for r in (1, 2, 3):
        h.observe_swap_out(r)
    h.observe_swap_in([3])
    h.observe_swap_out(3)
    h.observe_swap_in([3])
    assert recognize(h).kind is PatternKind.REPETITIVE
    assert [p.block for p in predict_next(h, h.outstanding, current_iv=0, leeway=0, depth=3)] == []


def test_classify_rules_and_c3():
    prof = ModelProfile("opt-13b", 629_278_720, 163_840)
    assert classify(32 * MIB, prof) is TransferClass.MODEL_WEIGHTS
    assert classify(25_298_944, prof) is TransferClass.MODEL_WEIGHTS
    assert classify(163_840, prof) is TransferClass.KV_CACHE
    assert classify(629_278_720, prof) is TransferClass.SMALL_IO  # defect C3
    assert classify(2048, prof) is TransferClass.SMALL_IO
    assert classify(256 * 1024, ModelProfile("x", 3 * 256 * 1024 + 100 * 1024, 4096),
                    PredictorConfig(chunk_bytes=256 * 1024)) is TransferClass.MODEL_WEIGHTS
    with pytest.raises(AmbiguousProfile):
        classify(5, ModelProfile("bad", 7, 7))
    with pytest.raises(ValueError):
        classify(0, prof)


def test_history_errors():
    h = SwapHistory()
    h.observe_swap_out(1)
    with pytest.raises(UnknownBlock):
        h.observe_swap_out(1)
    with pytest.raises(UnknownBlock):
        h.observe_swap_in([2])
    with pytest.raises(ValueError):
        h.observe_swap_in([])


@pytest.mark.parametrize("seed", range(40))
def test_incremental_matches_from_scratch(seed):
    """Random swap histories: the stateful Predictor (incremental streaks,
    groups and memoised cycle search) decides exactly as the from-scratch
    functions at every step."""
    rng = random.Random(seed)
    p = Predictor(ModelProfile("m", 1000, 10))
    on_gpu = set(range(1, 13))
    for _ in range(rng.randrange(30, 120)):
        r = rng.random()
        if r < 0.45 and on_gpu:
            b = rng.choice(sorted(on_gpu))
            on_gpu.discard(b)
            p.observe_swap_out(b)
        elif r < 0.85 and p.outstanding:
            out = sorted(p.outstanding)
            batch = rng.sample(out, rng.randrange(1, min(3, len(out)) + 1))
            p.observe_swap_in(batch)
            on_gpu.update(batch)
        else:
            p.observe_sync()
        h = p.history
        assert p.recognize() == recognize(h, p.config)
        assert h.groups_now() == outstanding_groups(h)
        for depth in (1, 2, 3):
            iv = rng.randrange(100)
            assert p.predict_batches(iv, 8, depth) == predict_batches(h, h.outstanding, iv, 8, depth, p.config)


def test_decision_log_lock_and_drop():
    p = Predictor(ModelProfile("m", 1000, 10))
    for b in (1, 2, 3):
        p.observe_swap_out(b)
    p.observe_swap_in([3]); p.observe_swap_out(3)
    p.observe_swap_in([3])
    assert p.decision_log[-1]["event"] == "lock" and p.decision_log[-1]["pattern"] == "repetitive"
