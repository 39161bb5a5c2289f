"""The bench's OPT-30B KV-swap comparison (config 3) alone, for A/B runs of
data-plane switches (SPPIPE_* env):  python tools/kv_ab.py [reps]"""
import os
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # as bench.py: no idle BLAS pool spinning
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload  # noqa: E402
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 7
cfg = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native",
                   reference_compat=False)
kv = workload.gen_adversarial_trace(
    workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
mem = prepare_memory(kv, cfg)
S = None
for name in os.environ.get("LD_PRELOAD", "").split(":"):
    if "sampler" in name:  # tools/native/sampler.c: sample the engine runs only
        import ctypes

        S = ctypes.CDLL(name)
        S.sampler_start()
        S.sampler_enable(0)
run_engine(kv, cfg, memory=mem)
run_plain_native(kv, cfg, memory=mem)
enc, pl = [], []
for _ in range(reps):
    if S:
        S.sampler_enable(1)
    enc.append(run_engine(kv, cfg, memory=mem).swap_gbs)
    if S:
        S.sampler_enable(0)
    pl.append(run_plain_native(kv, cfg, memory=mem).swap_gbs)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("SPPIPE_", "SPGCM_"))) or "default"
print(f"{env}: enc {max(enc):.2f} plain {max(pl):.2f} ratio {max(enc) / max(pl):.3f} "
      f"enc runs {[round(x, 1) for x in enc]}", flush=True)
r = run_engine(kv, cfg, memory=mem)
print("wall ms", round(r.wall_s * 1e3, 3))
print("plane stats", r.engine.plane_stats(), {k: v for k, v in r.engine.report().items() if k in ("syncs", "nops", "small_io_h2d", "small_io_d2h", "on_the_fly", "committed_sends", "deferred_decrypts")})
p = run_plain_native(kv, cfg, memory=mem)
print("plain wall ms", round(p.wall_s * 1e3, 3), "plain plane stats", p.engine.plane_stats())
