"""Multi-process (gloo, CPU) tests of the strip driver's host logic: strip
bounds, scene sharding and the D4 halo ring exchange. Each rank fuses its
strip with the ORACLE injected as the compute step (the exchange is what is
under test; the CUDA strip kernel is covered by tests/test_gpu_parity.py), and
the stitched result must equal the untiled oracle bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu_dwt as O
from paper_1803_00737_b200 import WaveletKind
from paper_1803_00737_b200 import strips

H, W, B = 96, 80, 3


def _scene():
    rng = np.random.default_rng(77)
    pan = rng.uniform(0, 255, (H, W)).astype(np.float32)
    ms = [rng.uniform(0, 255, (H // 2, W // 2)).astype(np.float32) for _ in range(B)]
    return pan, ms


def _oracle_compute(kind, pan, ms, halos):
    name = "haar" if kind is WaveletKind.HAAR else "daub4"
    if halos is None:
        return [torch.from_numpy(O.fuse_dwt(pan.numpy(), m.numpy(), name)) for m in ms]
    top, bot, mtop = halos
    win = torch.cat([top, pan, bot]).numpy()
    out = []
    for m, mt in zip(ms, mtop):
        mwin = torch.cat([mt, m, torch.zeros_like(mt)]).numpy()
        out.append(torch.from_numpy(O.fuse_dwt(win, mwin, name)[2:-2]))
    return out


def _worker(rank, world, port, kind_value, outdir, align):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pan, ms = _scene()
        r0, r1 = strips.strip_bounds(H, world, rank, align=align)
        p = torch.from_numpy(pan[r0:r1].copy())
        m = [torch.from_numpy(b[r0 // 2: r1 // 2].copy()) for b in ms]
        kind = WaveletKind(kind_value)
        out = strips.fuse_scene_strips(kind, p, m, compute=_oracle_compute)
        np.save(os.path.join(outdir, f"r{rank}.npy"), np.stack([o.numpy() for o in out]))
        mine = strips.shard(list(range(10)), rank, world)
        np.save(os.path.join(outdir, f"s{rank}.npy"), np.array(mine))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,align", [(2, 16), (3, 16), (4, 8)])
@pytest.mark.parametrize("kind", ["haar", "daub4"])
def test_strip_exchange_matches_untiled(tmp_path, world, align, kind):
    mp.spawn(_worker, args=(world, _free_port(), kind, str(tmp_path), align), nprocs=world,
             join=True)
    pan, ms = _scene()
    want = O.fuse(pan, ms, kind)
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(world)], axis=1)
    for b in range(B):
        assert np.array_equal(got[b], want[b]), (kind, world, b)
    owned = sorted(int(x) for r in range(world) for x in np.load(tmp_path / f"s{r}.npy"))
    assert owned == list(range(10))


def test_strip_bounds():
    assert strips.strip_bounds(65536, 8, 0) == (0, 8192)
    assert strips.strip_bounds(65536, 8, 7) == (57344, 65536)
    assert strips.strip_bounds(14000, 4, 3) == (10368, 14000)
    cover = [strips.strip_bounds(14000, 3, r) for r in range(3)]
    assert cover[0][0] == 0 and cover[-1][1] == 14000
    assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
    assert all((r1 - r0) % 2 == 0 for r0, r1 in cover)
    with pytest.raises(ValueError):
        strips.strip_bounds(64, 8, 0)


def test_single_rank_exchange_wraps_locally():
    pan = torch.arange(24, dtype=torch.float32).reshape(6, 4)
    ms = [torch.arange(6, dtype=torch.float32).reshape(3, 2)]
    top, bot, mtop = strips.exchange_halos(pan, ms)
    assert torch.equal(top, pan[-2:]) and torch.equal(bot, pan[:2])
    assert torch.equal(mtop[0], ms[0][-1:])
