"""Trace file format (workload.py:188-300): byte-identical JSONL, gzip
framing, parse errors and well-formedness rules."""
from __future__ import annotations

import pytest

from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.workload import (
    AppWriteEvent, ComputeEvent, SwapInRequest, SwapOut, SyncEvent, TraceFormatError, load_trace, save_trace,
    validate_trace,
)


@pytest.mark.parametrize("suffix", [".jsonl", ".jsonl.gz"])
def test_round_trip(tmp_path, suffix):
    tr = workload.gen_adversarial_trace(workload.gen_kvswap_trace(6, "lifo", kv_block_bytes=4096, seed=2), 0.5, 3)
    p = save_trace(tr, tmp_path / ("t" + suffix))
    back = load_trace(p)
    assert list(workload.trace_to_lines(back)) == list(workload.trace_to_lines(tr))
    assert back.swap_bytes() == tr.swap_bytes() and back.token_count() == tr.token_count()


def test_parse_errors(tmp_path):
    with pytest.raises(TraceFormatError):
        workload.parse_trace_lines([])
    with pytest.raises(TraceFormatError):
        workload.parse_trace_lines(['{"schema_version": 2}'])
    with pytest.raises(TraceFormatError):
        workload.parse_trace_lines(['{"oops": 1}'])
    good = list(workload.trace_to_lines(workload.gen_offload_trace(2, [1], 1, layer_bytes=64)))
    with pytest.raises(TraceFormatError):
        workload.parse_trace_lines(good + ['{"t": 9, "kind": "teleport"}'])
    with pytest.raises(TraceFormatError):
        load_trace(tmp_path / "missing.jsonl")


def test_validate_rules():
    tr = workload.gen_offload_trace(3, [1, 2], 1, layer_bytes=64)
    bad = [
        [SwapInRequest(5, 1), SyncEvent(1)],                  # time goes backwards
        [SwapOut(0, 1)],                                      # swap-out of a host-resident block
        [SwapInRequest(0, 1), SwapInRequest(0, 1)],           # swap-in of a block not outstanding
        [SwapInRequest(0, 1), ComputeEvent(0, 5)],            # compute inside an open batch
        [SwapInRequest(0, 1)],                                # trace ends inside a batch
        [AppWriteEvent(0, 1, 60, 10, 0)],                     # write outside the block
    ]
    for events in bad:
        t2 = workload.Trace(tr.header, events)
        with pytest.raises(TraceFormatError):
            validate_trace(t2)


def test_opt_shapes():
    assert workload.opt_layer_bytes("opt-13b") == 629_278_720
    assert workload.opt_layer_bytes("opt-66b") == 2_038_671_360
    assert workload.opt_kv_block_bytes("opt-30b") == 229_376
    tr = workload.gen_opt_offload_trace("opt-13b", [21], 1)
    sizes = sorted({b.nbytes for b in tr.header.blocks})
    assert sizes == [25_298_944, 32 * 1024 * 1024]


def test_jsonl_replay_cli_dry(tmp_path, capsys):
    """Reference-format JSONL traces replay through libsppipe from the
    command line (python -m paper_2411_03357_b200.replay), dispatched as one
    sp_pipe_replay call or event by event: the same decisions."""
    import json

    from paper_2411_03357_b200 import workload
    from paper_2411_03357_b200.replay import main

    tr = workload.gen_kvswap_trace(6, "lifo", kv_block_bytes=28672, parallel_size=2, seed=1)
    path = tmp_path / "kv.jsonl"
    workload.save_trace(tr, path)
    rows = []
    for dispatch in ("replay", "python"):
        assert main([str(path), "--plane", "dry", "--dispatch", dispatch, "--system", "specpipe"]) == 0
        rows.append(json.loads(capsys.readouterr().out.strip().splitlines()[-1]))
    assert rows[0] == rows[1] and rows[0]["error"] is None and rows[0]["data_msgs"] > 0
