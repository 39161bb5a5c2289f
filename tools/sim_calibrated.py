"""Recalibrate the reference simulator's CostModel (simulator.py:57-88) with
the B200 cells measured by tools/native/calibrate.cu and ask the reference's
own NoCc / SyncCc / SpecPipe sandwich what it predicts for the B200 data
plane.  Runs in the build container (it imports the
reference from /root/reference; nothing here is on the product path).

    python tools/sim_calibrated.py profiles/r1_calibrate_cells.json profiles/r1_sim_calibrated.json
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")


def fit(cells: list[dict]) -> dict:
    """CostModel fields from the measured cells.

    plain: fixed = API latency of the smallest copy; bandwidth = sustained
    32 MiB copies.  cc (B200 on-the-fly path, synchronous): fixed = latency of
    the smallest transfer; the plaintext crosses PCIe at the plain rate, so
    pcie_bw_cc = pcie_bw_plain; the crypto rate is what remains of the 32 MiB
    latency after the fixed cost and the wire time (one 'worker' = the GPU)."""
    by = {c["size"]: c for c in cells}
    small, big = by[min(by)], by[max(by)]
    bw_plain = big["plain_gbs"] * 1e9
    fixed_plain = small["plain_api_us"] * 1e-6
    fixed_cc = small["cc_api_us"] * 1e-6
    wire = max(by) / bw_plain
    crypto_s = big["cc_api_us"] * 1e-6 - fixed_cc - wire
    return {"pcie_bw_plain": bw_plain, "pcie_bw_cc": bw_plain, "crypto_bw_per_worker": max(by) / crypto_s,
            "fixed_overhead_plain": fixed_plain, "fixed_overhead_cc": fixed_cc}


def main(cells_path: str, out_path: str, measured_ratio: float | None = None) -> None:
    from specpipe import simulator as sim
    from specpipe import workload as ref_workload

    cells = json.load(open(cells_path))["cells"]
    params = fit(cells)
    cost = sim.CostModel(**params)
    report = {"fit": params, "cells": cells,
              "h100_reference_cells": {"latency_us": {k.value: v for k, v in sim.REFERENCE_LATENCY_US.items()},
                                       "throughput_gbs": {k.value: v for k, v in sim.REFERENCE_THROUGHPUT_GBS.items()}}}
    # the reference's sandwich on the bench's OPT-66B offload shape (2 of the
    # offloaded layers, 61 x 32 MiB chunks; 2 iterations keep the pure-Python
    # simulator within minutes)
    from paper_2411_03357_b200 import workload

    tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2)
    lines = list(workload.trace_to_lines(tr))
    rtr = ref_workload.parse_trace_lines(lines)
    preds = {}
    for system, workers in (("nocc", 1), ("synccc", 1), ("specpipe", 1)):
        t = time.time()
        m = sim.run(rtr, sim.SimConfig(system=sim.SystemKind(system), workers=workers, cost=cost))
        preds[system] = {"throughput_gbs": m.throughput_bytes_per_s / 1e9, "makespan_ms": m.makespan_ns / 1e6,
                         "hit_rate": m.hit_rate, "nops": m.nop_count, "sim_wall_s": round(time.time() - t, 1)}
        print(system, preds[system], flush=True)
    report["prediction_opt66b"] = preds
    report["predicted_specpipe_vs_nocc"] = preds["specpipe"]["throughput_gbs"] / preds["nocc"]["throughput_gbs"]
    report["predicted_synccc_vs_nocc"] = preds["synccc"]["throughput_gbs"] / preds["nocc"]["throughput_gbs"]
    if measured_ratio is not None:
        report["measured_specpipe_vs_nocc"] = measured_ratio
    json.dump(report, open(out_path, "w"), indent=1)
    print(json.dumps({k: v for k, v in report.items() if k.startswith(("pred", "meas", "fit"))}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
