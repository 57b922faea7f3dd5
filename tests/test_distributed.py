"""Row-sharded multi-GPU Gram, host logic on CPU: world_size 2 over gloo.

The per-rank compute is injected (the CPU oracle as a stand-in for the
rank's GPU) so the partitioning, the collective and the assembly are exercised
exactly as `bench.py --gpus N` runs them over NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_07145_b200.distributed import row_blocks, sharded_gram, triangle_row_blocks


def test_row_blocks_cover_and_balance():
    for n in (1, 7, 64, 1000):
        for w in (1, 2, 3, 8):
            b = row_blocks(n, w)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(w - 1))
            t = triangle_row_blocks(n, w)
            assert t[0][0] == 0 and t[-1][1] == n
            assert all(t[r][1] == t[r + 1][0] for r in range(w - 1))
    pairs = [sum(1000 - i for i in range(a, b)) for a, b in triangle_row_blocks(1000, 8)]
    assert max(pairs) - min(pairs) <= 2 * 1000  # within two rows of perfect balance


def _oracle_compute(X, Y, cfg, r0, r1, precision, K_full):
    from oracle import sigkern_oracle as O
    Xn = X.numpy()
    if Y is None:
        # symmetric: this rank's triangle rows and their mirror into the zeroed full K
        full = O.gram(Xn, None, M=cfg.n_levels, p=cfg.effective_order,
                      normalization=cfg.normalization)
        for i in range(r0, r1):
            K_full[i, i:] = torch.from_numpy(full[i, i:])
            K_full[i:, i] = torch.from_numpy(full[i:, i])
        return K_full
    full = O.gram(Xn, Y.numpy(), M=cfg.n_levels, p=cfg.effective_order,
                  normalization=cfg.normalization)
    return torch.from_numpy(full[r0:r1])


def _worker(rank, world, port, sym, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_07145_b200 import KernelConfig, SeedStream, gen_brownian
        X = torch.from_numpy(gen_brownian(7, 6, 2, SeedStream(3)).data)
        Y = None if sym else torch.from_numpy(gen_brownian(5, 5, 2, SeedStream(4)).data)
        cfg = KernelConfig(n_levels=3, normalization="levelwise")
        K = sharded_gram(X, Y, cfg, compute=_oracle_compute)
        out_q.put((rank, K.numpy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("sym", [False, True])
def test_sharded_gram_gloo_world2(sym):
    from oracle import sigkern_oracle as O
    from paper_2501_07145_b200 import SeedStream, gen_brownian
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sym, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = gen_brownian(7, 6, 2, SeedStream(3)).data
    Y = None if sym else gen_brownian(5, 5, 2, SeedStream(4)).data
    want = O.gram(X, Y, M=3, p=1, normalization="levelwise")
    for r in range(2):
        assert res[r].shape == want.shape
        assert np.array_equal(res[r], want)  # every entry has exactly one contributor


def _gpu_worker(rank, world, port, sym, out_q):
    """sharded_gram with its real compute: both ranks on cuda:0, gloo collectives."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_07145_b200 import KernelConfig, SeedStream, gen_brownian
        torch.cuda.set_device(0)
        X = torch.from_numpy(gen_brownian(37, 40, 5, SeedStream(3)).data).cuda()
        Y = None if sym else torch.from_numpy(gen_brownian(29, 33, 5, SeedStream(4)).data).cuda()
        cfg = KernelConfig(n_levels=4, normalization="levelwise")
        K = sharded_gram(X, Y, cfg)
        out_q.put((rank, K.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("sym", [False, True])
def test_sharded_gram_gpu_world2_bitwise(sym):
    """The row-sharded Gram with the rank's GPU compute equals the single-GPU
    Gram bit for bit (cross: row blocks; symmetric: paired blocks + mirror)."""
    from paper_2501_07145_b200 import KernelConfig, SeedStream, gen_brownian
    from paper_2501_07145_b200.kernels import sig_kernel_gram
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, sym, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = gen_brownian(37, 40, 5, SeedStream(3)).data
    Y = None if sym else gen_brownian(29, 33, 5, SeedStream(4)).data
    want = sig_kernel_gram(X, Y, cfg=KernelConfig(n_levels=4, normalization="levelwise"))
    for r in range(2):
        assert np.array_equal(res[r], want)
    if sym:
        assert np.array_equal(res[0], res[0].T)


def test_paired_row_blocks_balance():
    from paper_2501_07145_b200.distributed import paired_row_blocks
    for n in (1, 5, 64, 1000, 8192):
        for w in (1, 2, 3, 8):
            blocks = paired_row_blocks(n, w)
            rows = sorted(r for rb in blocks for r in rb if r[1] > r[0])
            assert rows[0][0] == 0 and rows[-1][1] == n
            assert all(rows[k][1] == rows[k + 1][0] for k in range(len(rows) - 1))
    pairs = [sum(sum(8192 - i for i in range(a, b)) for a, b in rb)
             for rb in paired_row_blocks(8192, 8)]
    assert max(pairs) - min(pairs) <= 8192 * 2


def _weak_worker(rank, world, port, n, out_q):
    """bench.py's multi-GPU partition: rank r owns sequences [r*n, (r+1)*n) of X
    (prefix-stable generator) and evaluates its row block of K(X, Y); no collective
    in the computation (the gather below only verifies the result)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sigkern_oracle as O
        from paper_2501_07145_b200 import SeedStream, gen_brownian
        Xr = gen_brownian(n, 6, 2, SeedStream(1), start=rank * n).data
        Y = gen_brownian(4, 6, 2, SeedStream(2)).data
        Kr = torch.from_numpy(O.gram(Xr, Y, M=3, p=1, normalization="levelwise"))
        parts = [torch.empty_like(Kr) for _ in range(world)]
        dist.all_gather(parts, Kr)
        out_q.put((rank, torch.cat(parts).numpy()))
    finally:
        dist.destroy_process_group()


def test_weak_scaling_partition_gloo_world2():
    from oracle import sigkern_oracle as O
    from paper_2501_07145_b200 import SeedStream, gen_brownian
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 3
    procs = [ctx.Process(target=_weak_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = gen_brownian(2 * n, 6, 2, SeedStream(1)).data
    Y = gen_brownian(4, 6, 2, SeedStream(2)).data
    want = O.gram(X, Y, M=3, p=1, normalization="levelwise")
    assert np.array_equal(res[0], want) and np.array_equal(res[1], want)
