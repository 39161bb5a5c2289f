"""A/B of data-plane switches (SPPIPE_* env, read once per process) on the
config-5 offload trace at a few block sizes and on the config-3 KV trace,
swap-only and with the model's compute: run once per setting, compare the
printed rows.   python tools/ab_switch.py [block_kib,...]"""
import json
import os
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03357_b200 import workload  # noqa: E402
from paper_2411_03357_b200.replay import ReplayConfig, prepare_memory, run_engine, run_plain_native  # noqa: E402

sizes = ([int(x) for x in sys.argv[1].split(",") if x and x != "none"] if len(sys.argv) > 1
         else [64, 1024, 32768, 262144])
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("SPPIPE_", "SPGCM_", "AB_CRYPTO"))) or "default"
reps = int(os.environ.get("AB_REPS", "2"))


def best(fn):
    return max(fn().swap_gbs for _ in range(reps))


def arms(tr, base):
    if os.environ.get("AB_CRYPTO_SMS"):  # SM budget of the crypto launches (ReplayConfig.crypto_sms)
        base = replace(base, crypto_sms=int(os.environ["AB_CRYPTO_SMS"]))
    out = {}
    for comp in (False, True):
        c = replace(base, compute=comp)
        mem = prepare_memory(tr, c)
        run_plain_native(tr, c, memory=mem)
        run_engine(tr, c, memory=mem)
        p = best(lambda: run_plain_native(tr, c, memory=mem))
        e = best(lambda: run_engine(tr, c, memory=mem))
        out["compute" if comp else "swap_only"] = {"plain": round(p, 2), "specpipe": round(e, 2), "ratio": round(e / p, 4)}
        del mem
    return out


for kib in sizes:
    blk = kib << 10
    msg = min(blk, 32 << 20)
    tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=2, chunk_bytes=blk)
    base = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native",
                        chunk_bytes=msg, predictor_chunk_bytes=msg, reference_compat=False)
    print(json.dumps({"env": env, "block_kib": kib, **arms(tr, base)}), flush=True)
if os.environ.get("AB_175B"):  # the bench's OPT-175B 4-bit leg (2 x 906 MB layers, 2 iterations)
    tr = workload.gen_opt_offload_trace("opt-175b", [1, 2], iterations=2, seed=0, quant_bits=4)
    base = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native")
    print(json.dumps({"env": env, "trace": "opt175b_4bit", **arms(tr, base)}), flush=True)
if os.environ.get("AB_66B"):  # the bench's OPT-66B leg (8 iterations)
    tr = workload.gen_opt_offload_trace("opt-66b", [1, 2], iterations=8, seed=0)
    base = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native")
    print(json.dumps({"env": env, "trace": "opt66b_8it", **arms(tr, base)}), flush=True)
kv = workload.gen_adversarial_trace(
    workload.gen_kvswap_trace(48, "lifo", kv_block_bytes=229_376, parallel_size=4, seed=0), 0.25, seed=8)
reps = 5
base = ReplayConfig(system="specpipe", plane="gpu", record_stream=False, fill="fast", engine="native",
                    reference_compat=False)
print(json.dumps({"env": env, "trace": "kv", **arms(kv, base)}), flush=True)
