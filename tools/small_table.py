"""bench.py's small-message table alone (graph-replayed device time per
launch), one line per case, prefixed with the SPGCM_* environment: for
launch-policy A/B runs (python tools/small_table.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_03357_b200.gcm import GcmContext  # noqa: E402

env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SPGCM_")) or "default"
t = bench.small_message_table(GcmContext(bytes(range(32))), torch.device("cuda:0"))
for r in t["rows"]:
    print(f"{env:50s} {r['case']:18s} {r.get('us_per_launch', r.get('error'))}", flush=True)
