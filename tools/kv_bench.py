"""OPT-30B KV-swap (config 3 shape) through the engine vs plain swaps, and the
control-plane-only cost (dry plane)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload
from paper_2411_03357_b200.replay import ReplayConfig, run_engine, run_plain, run_plain_native
plane = sys.argv[1] if len(sys.argv) > 1 else "gpu"
for pol in ("lifo", "fifo"):
    base = workload.gen_kvswap_trace(48, pol, kv_block_bytes=229_376, parallel_size=4, seed=0)
    for rate in (0.0, 0.25):
        tr = workload.gen_adversarial_trace(base, rate, seed=8) if rate else base
        dry = run_engine(tr, ReplayConfig(plane="dry", reference_compat=False))
        line = f"{pol} rate={rate} events={len(tr.events)} swap={tr.swap_bytes()/1e6:.1f}MB dry {dry.wall_s*1e3:.1f} ms"
        if plane == "gpu":
            run_engine(tr, ReplayConfig(plane="gpu", reference_compat=False, fill="fast"))
            enc = run_engine(tr, ReplayConfig(plane="gpu", reference_compat=False, fill="fast"))
            ncfg = ReplayConfig(plane="gpu", reference_compat=False, fill="fast", engine="native")
            run_engine(tr, ncfg)
            nat = min((run_engine(tr, ncfg) for _ in range(3)), key=lambda r: r.wall_s)
            run_plain(tr, fill="fast")
            pl = min((run_plain(tr, fill="fast") for _ in range(3)), key=lambda r: r.wall_s)
            run_plain_native(tr, ncfg)
            pn = min((run_plain_native(tr, ncfg) for _ in range(3)), key=lambda r: r.wall_s)
            line += (f" | py-engine {enc.wall_s*1e3:.1f} ms ({enc.swap_gbs:.2f} GB/s) native {nat.wall_s*1e3:.1f} ms "
                     f"({nat.swap_gbs:.2f} GB/s) plain(py) {pl.wall_s*1e3:.1f} ms ({pl.swap_gbs:.2f} GB/s) "
                     f"plain(native) {pn.wall_s*1e3:.1f} ms ({pn.swap_gbs:.2f} GB/s)")
        print(line, flush=True)
