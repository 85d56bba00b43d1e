"""Peer-memory halos (strips.PeerHalos): two processes, each fusing one row
strip of a D4 scene, read their neighbour's halo rows through CUDA IPC
mappings instead of exchanging them. Both processes share the one GPU of the
test box (the IPC mapping is then same-device; on the 8-GPU node it is an
NVLink peer mapping); the kernels only READ the neighbour's static inputs, so
nothing waits on anything. The stitched result must equal the untiled
fusion bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

H, W, B = 256, 1040, 3


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1803_00737_b200 as wf
        from paper_1803_00737_b200 import strips, synth

        torch.cuda.set_device(0)
        r0, r1 = strips.strip_bounds(H, world, rank, align=2)
        pan = torch.empty((r1 - r0, W), device="cuda")
        synth.device_plane(pan, 7, 0, row0=r0)
        ms = []
        for b in range(B):
            t = torch.empty(((r1 - r0) // 2, W // 2), device="cuda")
            synth.device_plane(t, 7, 1 + b, row0=r0 // 2)
            ms.append(t)
        torch.cuda.synchronize()
        dist.barrier()  # every strip's inputs exist before anyone maps them
        halos = strips.PeerHalos(pan, ms)
        out = strips.fuse_strip(wf.WaveletKind.DAUB4, pan, ms, halos)
        # the reference-exact strip kernel reads the same peer halo rows
        ex = strips.fuse_strip(wf.WaveletKind.DAUB4, pan, ms, halos, exact=True)
        torch.cuda.synchronize()
        dist.barrier()  # neighbours are done reading before mappings go away
        halos.close()
        np.save(os.path.join(outdir, f"r{rank}.npy"), np.stack([o.cpu().numpy() for o in out]))
        np.save(os.path.join(outdir, f"x{rank}.npy"), np.stack([o.cpu().numpy() for o in ex]))
    finally:
        dist.destroy_process_group()


def test_peer_halos_two_processes(tmp_path):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    import paper_1803_00737_b200 as wf
    from paper_1803_00737_b200 import synth

    pan = torch.empty((H, W), device="cuda")
    synth.device_plane(pan, 7, 0)
    ms = []
    for b in range(B):
        t = torch.empty((H // 2, W // 2), device="cuda")
        synth.device_plane(t, 7, 1 + b)
        ms.append(t)
    want = [o.cpu().numpy() for o in wf.fuse(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4))]
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(2)], axis=1)
    for b in range(B):
        assert np.array_equal(got[b], want[b])
    # exact strips across ranks == the exact whole scene (the reference's bits)
    want_x = [o.cpu().numpy() for o in wf.fuse(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4),
                                               exact=True)]
    got_x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(2)], axis=1)
    for b in range(B):
        assert np.array_equal(got_x[b], want_x[b])


def test_peer_halos_single_rank_wraps_locally():
    import paper_1803_00737_b200 as wf
    from paper_1803_00737_b200 import strips

    g = torch.Generator(device="cuda").manual_seed(1)
    pan = torch.rand((128, 520), generator=g, device="cuda") * 255
    ms = [torch.rand((64, 260), generator=g, device="cuda") * 255 for _ in range(2)]
    got = strips.fuse_strip(wf.WaveletKind.DAUB4, pan, ms, strips.PeerHalos(pan, ms))
    want = wf.fuse(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4))
    for a, b in zip(got, want):
        assert torch.equal(a, b)
