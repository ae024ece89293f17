"""Host side of the x-slab decomposition on CPU: slab ownership (include/sog.h rule) and the
particle redistribution helper over torch.distributed with the gloo backend, world size 2."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2412_04595_b200.sog import redistribute, slab_owner  # noqa: E402
from synth import config_system  # noqa: E402


def test_slab_owner_rule():
    L = 215.0
    for R in (1, 2, 3, 8):
        x = np.concatenate([np.linspace(-L / 2, L / 2, 10001), -L / 2 + L * np.arange(R + 1) / R,
                            np.array([-L / 2 - 1e-9, L / 2 + 3.0, 1e3])])
        r = slab_owner(x, L, R)
        xc = x - L * np.floor((x + L / 2) / L)
        xc = np.where(xc >= L / 2, xc - L, xc)
        lo = -L / 2 + L * r / R
        hi = np.where(r + 1 == R, L / 2, -L / 2 + L * (r + 1) / R)
        assert np.all((xc >= lo) & (xc < hi)), R
        assert np.all((r >= 0) & (r < R))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    xyz, q, L = config_system("c5", N=3000)
    # every rank starts with an arbitrary (interleaved) share of the system
    mine = np.arange(rank, len(q), ws)
    x, qq, origin = redistribute(torch.from_numpy(xyz[mine]), torch.from_numpy(q[mine]), L)
    owner = slab_owner(x[:, 0].numpy(), L[0], ws)
    glob = np.array([np.arange(int(r), len(q), ws)[int(i)] for r, i in origin.numpy()])
    ok = bool(np.all(owner == rank)) and np.allclose(x.numpy(), xyz[glob]) and np.allclose(qq.numpy(), q[glob])
    n = torch.tensor([len(qq)])
    dist.all_reduce(n)
    q_out.put((rank, ok, int(n.item())))
    dist.destroy_process_group()


def test_redistribute_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, qo)) for r in range(2)]
    for p in ps:
        p.start()
    res = [qo.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(n == 3000 for _, _, n in res), res
