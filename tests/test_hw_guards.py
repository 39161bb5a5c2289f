"""Hardware write guards (libspguard): a store that bypasses
HostMemory.write into a speculatively encrypted range must invalidate the
record, so the stale ciphertext is never committed.  Run in a subprocess:
the check installs a SIGSEGV handler."""
from __future__ import annotations

import os
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent('''
    import sys
    sys.path.insert(0, %r)
    from paper_2411_03357_b200 import guards
    from paper_2411_03357_b200.channel import new_channel
    from paper_2411_03357_b200.engine import CopyRequest, Engine, EngineConfig
    from paper_2411_03357_b200.memory import HostMemory, ModelLayer, prng_fill
    from paper_2411_03357_b200.predictor import Prediction, Predictor, TransferClass
    from paper_2411_03357_b200.validator import RecordState

    mem = HostMemory(pinned=False, hw_guards=True)
    cpu, gpu = new_channel(seed=1)
    b = mem.alloc(ModelLayer(1), 256 * 1024, prng_fill(3))
    c = mem.alloc(ModelLayer(2), 256 * 1024, prng_fill(4))
    eng = Engine(mem, cpu, gpu, Predictor.scripted([[Prediction(b.id, 0, 0), Prediction(c.id, 1, 0)]], {b.id, c.id}),
                 EngineConfig(leeway=0, plane="dry"))
    eng.speculate_tick()   # queue the encrypt-ahead
    eng.speculate_tick()   # the next entry point seals, labels and guards it
    assert guards.active() == 2, guards.active()
    rec_b = next(r for r in eng.validator.records.values() if r.block_id == b.id)
    # 1) a direct store (numpy, no HostMemory.write) into b's guarded pages
    b.data[100000] ^= 0xFF
    assert guards.faults() == 1
    # 2) the next engine entry turns it into an invalidation
    h = eng.copy_h2d(CopyRequest("h2d", b.base, b.len, TransferClass.MODEL_WEIGHTS, block_id=b.id))
    assert rec_b.state is RecordState.INVALIDATED, rec_b.state
    assert h.verdict.value == "stale", h.verdict          # sent on the fly with the new bytes
    assert eng.report()["write_faults"] == 1
    # c is untouched: still a HIT
    h2 = eng.copy_h2d(CopyRequest("h2d", c.base, c.len, TransferClass.MODEL_WEIGHTS, block_id=c.id))
    assert h2.verdict.value == "hit", h2.verdict
    # 3) released guards leave the pages writable; API writes never trap
    c.data[7] = 1
    mem.write(b.id, 0, b"xyz")
    assert guards.active() == 0
    eng.finish()
    print("hw guards ok", guards.faults())
''' % ROOT)


def test_hw_guard_invalidates_on_direct_store():
    out = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "hw guards ok 1" in out.stdout


def test_hw_guard_library_exports():
    import re

    from paper_2411_03357_b200 import guards

    text = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "spguard.h")).read(), flags=re.S)
    names = set(re.findall(r"\b(spg_[a-z_]+)\s*\(", text))
    assert names == set(guards.SYMBOLS)
    lib = guards.lib()
    for n in names:
        assert hasattr(lib, n)


GPU_SCRIPT = SCRIPT.replace("HostMemory(pinned=False, hw_guards=True)", "HostMemory(pinned=True, hw_guards=True)") \
                   .replace('plane="dry"', 'plane="gpu"')


import pytest  # noqa: E402


@pytest.mark.gpu
def test_hw_guard_on_pinned_memory_gpu():
    """Same check on page-locked (cudaHostAlloc) blocks with the B200 plane:
    mprotect works on pinned pages and DMA is unaffected."""
    out = subprocess.run([sys.executable, "-c", GPU_SCRIPT], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "hw guards ok 1" in out.stdout


NATIVE_SCRIPT = textwrap.dedent('''
    import sys
    sys.path.insert(0, %r)
    from paper_2411_03357_b200 import guards
    from paper_2411_03357_b200.channel import new_channel
    from paper_2411_03357_b200.engine import CopyRequest, Engine, EngineConfig
    from paper_2411_03357_b200.memory import HostMemory, ModelLayer, prng_fill
    from paper_2411_03357_b200.predictor import ModelProfile, Predictor, TransferClass

    W = TransferClass.MODEL_WEIGHTS
    mem = HostMemory(pinned=PINNED, hw_guards=True)
    cpu, gpu = new_channel(seed=1)
    pred = Predictor(ModelProfile("m", 256 * 1024, 4096))
    eng = Engine(mem, cpu, gpu, pred, EngineConfig(leeway=0, plane=PLANE))
    blocks = [mem.alloc(ModelLayer(i), 256 * 1024, prng_fill(i)) for i in range(4)]
    for b in blocks:
        pred.observe_swap_out(b.id)
    req = lambda b: CopyRequest("h2d", b.base, b.len, W, block_id=b.id)
    # two FIFO batches lock the pattern; the sync after the second queues
    # encrypt-ahead of block 3, labeled (and guarded) at the next entry
    for b in blocks[:2]:
        eng.copy_h2d(req(b))
        eng.sync()
        eng.copy_d2h(CopyRequest("d2h", b.base, b.len, W, block_id=b.id))
    assert guards.active() >= 1, guards.active()
    target = blocks[2]
    target.data[100000] ^= 0xFF          # a direct store: no app_write, no HostMemory.write
    assert guards.faults() == 1
    h = eng.copy_h2d(req(target))        # the entry point turns the trap into an invalidation
    assert h.verdict.value == "stale", h.verdict
    assert eng.report()["write_faults"] == 1
    eng.sync()
    eng.finish()
    assert guards.active() == 0
    print("native hw guards ok", guards.faults())
''' % ROOT)


def test_hw_guard_from_learned_prediction():
    script = NATIVE_SCRIPT.replace("PINNED", "False").replace("PLANE", '"dry"')
    out = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "native hw guards ok 1" in out.stdout


@pytest.mark.gpu
def test_hw_guard_from_learned_prediction_gpu():
    script = NATIVE_SCRIPT.replace("PINNED", "True").replace("PLANE", '"gpu"')
    out = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "native hw guards ok 1" in out.stdout


RACE_SCRIPT = textwrap.dedent('''
    import ctypes, mmap, sys, threading
    sys.path.insert(0, %r)
    import numpy as np
    from paper_2411_03357_b200 import guards

    PAGE = mmap.PAGESIZE
    L = guards.lib()
    m = mmap.mmap(-1, 8 * PAGE)
    buf = np.frombuffer(m, dtype=np.uint8)
    base = buf.ctypes.data
    assert base %% PAGE == 0

    # (1) partial tail page: protected only when the caller owns it
    u0 = guards.uncovered()
    guards.protect(base, 2 * PAGE + 100, 1)              # tail page left writable
    assert guards.uncovered() == u0 + 1
    ctypes.memset(base + 2 * PAGE + 50, 7, 1)             # no fault: page not covered
    assert guards.faults() == 0
    guards.release(1)
    guards.protect(base, 2 * PAGE + 100, 2, guards.HEAD_OWNED | guards.TAIL_OWNED)
    assert guards.uncovered() == u0 + 1
    ctypes.memset(base + 2 * PAGE + 50, 8, 1)             # traps: the tail page is the block's
    assert guards.faults() == 1 and guards.drain() == [2]
    guards.release(2)

    # (2) many threads storing into one guard at once, and a release racing
    #     the stores: every store must retry and land, none may crash
    n_rounds, n_threads = 200, 8
    for r in range(n_rounds):
        guards.protect(base + 4 * PAGE, 2 * PAGE, 100 + r)
        go = threading.Event()
        def store(k):
            go.wait()
            ctypes.memset(base + 4 * PAGE + 64 * k, r & 0xFF, 64)   # ctypes drops the GIL
        ts = [threading.Thread(target=store, args=(k,)) for k in range(n_threads)]
        if r %% 2:
            ts.append(threading.Thread(target=lambda: (go.wait(), guards.release(100 + r))))
        for t in ts:
            t.start()
        go.set()
        for t in ts:
            t.join()
        guards.release(100 + r)
        assert all(buf[4 * PAGE + 64 * k] == (r & 0xFF) for k in range(n_threads))
    drained = guards.drain()
    assert len(drained) <= n_rounds and guards.active() == 0
    print("guard race ok", guards.faults())
''' % ROOT)


def test_hw_guard_tail_page_and_concurrent_stores():
    """partial tail pages of page-owned blocks are protected; a
    store racing another thread's fault or a release retries instead of
    reaching SIG_DFL."""
    out = subprocess.run([sys.executable, "-c", RACE_SCRIPT], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "guard race ok" in out.stdout
