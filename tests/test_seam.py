"""INTEGRATION.md §2, executed: the UNCHANGED reference package (installed
from /root/reference into baseline/_ref) with only its three crypto names
rebound to libspgcm (paper_2411_03357_b200.seam) runs the reference
simulator's engine over the golden traces and reproduces the goldens that
the reference produced with its own `cryptography` AES-GCM: sent logs,
actions, report, decision log, errors and delivered plaintext digests.
Skipped when baseline/_ref is absent."""
from __future__ import annotations

import json
import os
import sys
import tempfile

import pytest

from tests.test_engine_parity import GOLD, action_tuple, make_trace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _specpipe():
    if not os.path.isdir(os.path.join(REF, "specpipe")):
        pytest.skip("baseline/_ref (the reference install) is absent")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import specpipe
    import specpipe.engine  # noqa: F401
    import specpipe.simulator  # noqa: F401

    return specpipe


def test_seam_rebinds_the_three_names():
    specpipe = _specpipe()
    from paper_2411_03357_b200 import seam

    before = (specpipe.channel.encrypt_at, specpipe.channel.decrypt_at, specpipe.engine.encrypt_at)
    old = seam.install(specpipe)
    try:
        assert old == before
        now = (specpipe.channel.encrypt_at, specpipe.channel.decrypt_at, specpipe.engine.encrypt_at)
        assert all(a is not b for a, b in zip(now, before))
        assert now[0] is now[2]
    finally:
        seam.uninstall(specpipe, old)
    assert (specpipe.channel.encrypt_at, specpipe.channel.decrypt_at, specpipe.engine.encrypt_at) == before


def _reference_trace(specpipe, params):
    from paper_2411_03357_b200 import workload

    tr = make_trace(params)
    with tempfile.NamedTemporaryFile("w", suffix=".jsonl", delete=False) as fh:
        fh.write("\n".join(workload.trace_to_lines(tr)) + "\n")
    try:
        return specpipe.workload.load_trace(fh.name)
    finally:
        os.unlink(fh.name)


@pytest.mark.gpu
def test_unchanged_reference_engine_on_libspgcm_gpu():
    specpipe = _specpipe()
    from paper_2411_03357_b200 import _native, seam

    sim, D = specpipe.simulator, specpipe.channel.Direction
    calls = {"seal": 0, "open": 0}
    old = seam.install(specpipe)
    enc, dec = specpipe.channel.encrypt_at, specpipe.channel.decrypt_at

    def counting_enc(*a, **k):
        calls["seal"] += 1
        return enc(*a, **k)

    def counting_dec(*a, **k):
        calls["open"] += 1
        return dec(*a, **k)

    specpipe.channel.encrypt_at = specpipe.engine.encrypt_at = counting_enc
    specpipe.channel.decrypt_at = counting_dec
    launches0 = _native.launch_count()
    try:
        for case in GOLD:
            if case["name"].startswith("full_offload"):
                continue  # 1.2 GB through the reference's Python engine: the native path covers it
            rt = _reference_trace(specpipe, case["params"])
            kind = {"specpipe": sim.SystemKind.SPECPIPE, "synccc": sim.SystemKind.SYNCCC}[case["system"]]
            rp = sim._Replay(rt, sim.SimConfig(system=kind, record_stream=True))
            try:
                rp.run()
                err = None
            except Exception as exc:
                err = f"{type(exc).__name__}: {exc}"
            eng = rp.engine
            assert err == case["error"], case["name"]
            assert [list(x) for x in eng.cpu.channel.sent_log(D.HOST_TO_DEVICE)] == case["sent_h2d"]
            assert [list(x) for x in eng.cpu.channel.sent_log(D.DEVICE_TO_HOST)] == case["sent_d2h"]
            assert [action_tuple(a) for a in eng.actions] == case["actions"], case["name"]
            assert json.loads(json.dumps(eng.report())) == case["report"], case["name"]
            assert eng.predictor.decision_log == case["decision_log"], case["name"]
            assert [list(d) for d in eng.delivered] == case["delivered"], case["name"]
            assert [list(d) for d in eng.d2h_stream] == case["d2h_stream"], case["name"]
    finally:
        seam.uninstall(specpipe, old)
    assert calls["seal"] > 100 and calls["open"] > 100
    assert _native.launch_count() - launches0 >= calls["seal"] + calls["open"]  # every call ran a k_gcm launch
