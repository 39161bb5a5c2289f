"""k_xfer, the data plane's SM-driven host<->device transfer of small copies
(csrc/sppipe.cu): byte-identical to the source for both
directions, every alignment class (16 B vector body, byte path, job tails),
zero-length jobs and jobs split across many 16 KiB pieces.  It stands in for
cudaMemcpyAsync, so the oracle is the source bytes themselves."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch

    torch.cuda.set_device(0)
    from paper_2411_03357_b200 import _native

    return _native.load_sppipe()


def _run(lib, dsts, srcs, lens):
    n = len(lens)
    D = (ctypes.c_void_p * n)(*dsts)
    S = (ctypes.c_void_p * n)(*srcs)
    L = (ctypes.c_uint64 * n)(*lens)
    rc = lib.sp_test_xfer(n, D, S, L)
    assert rc == 0, lib.sp_pipe_last_error()


@pytest.mark.parametrize("h2d", [True, False])
def test_xfer_alignments_and_sizes(lib, h2d):
    import torch

    rng = np.random.default_rng(7 + h2d)
    host = torch.empty(8 << 20, dtype=torch.uint8, pin_memory=True)
    dev = torch.zeros(8 << 20, dtype=torch.uint8, device="cuda")
    src_t, dst_t = (host, dev) if h2d else (dev, host)
    payload = torch.from_numpy(rng.integers(0, 256, 8 << 20, dtype=np.uint8))
    if h2d:
        host.copy_(payload)
    else:
        dev.copy_(payload.cuda())
        host.zero_()
    # (src offset, dst offset, length): aligned, misaligned, mixed, tails, empty, multi-piece
    cases = [(0, 0, 229376), (16, 32, 65536 + 5), (3, 3, 1000), (5, 9, 4097), (0, 7, 77), (1, 0, 1),
             (4096, 8192, 0), (32, 48, 3 * 16384 + 15), (7, 1, 100_003), (64, 64, 2 << 20)]
    dsts, srcs, lens, spans = [], [], [], []
    s_cur, d_cur = 0, 0
    for so, do, n in cases:
        s_at, d_at = s_cur + so, d_cur + do
        srcs.append(src_t.data_ptr() + s_at)
        dsts.append(dst_t.data_ptr() + d_at)
        lens.append(n)
        spans.append((s_at, d_at, n))
        s_cur = (s_at + n + 4095) & ~4095
        d_cur = (d_at + n + 4095) & ~4095
    _run(lib, dsts, srcs, lens)
    torch.cuda.synchronize()
    got = dst_t.cpu().numpy() if not h2d else dev.cpu().numpy()
    want = payload.numpy()
    for s_at, d_at, n in spans:
        assert np.array_equal(got[d_at:d_at + n], want[s_at:s_at + n]), (s_at, d_at, n)
    # nothing written outside the jobs
    mask = np.zeros(got.size, dtype=bool)
    for _, d_at, n in spans:
        mask[d_at:d_at + n] = True
    assert not got[~mask].any()


def test_xfer_many_jobs(lib):
    """128 jobs (a full launch) of KV-block size, host -> device."""
    import torch

    n, blk = 128, 16384 + 48
    host = torch.randint(0, 256, (n * blk,), dtype=torch.uint8).pin_memory()
    dev = torch.zeros(n * blk, dtype=torch.uint8, device="cuda")
    _run(lib, [dev.data_ptr() + i * blk for i in range(n)], [host.data_ptr() + i * blk for i in range(n)], [blk] * n)
    torch.cuda.synchronize()
    assert torch.equal(dev.cpu(), host)


def test_xfer_rejects_bad_counts(lib):
    L = (ctypes.c_uint64 * 1)(1)
    assert lib.sp_test_xfer(129, None, None, L) != 0
    assert lib.sp_test_xfer(0, None, None, None) == 0
