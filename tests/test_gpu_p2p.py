"""K1 with the all-gather fused into its epilogue (cpsj_minhash_sketch_multi
+ CUDA IPC exchange buffers, distributed.PeerArrays / embed_sharded_p2p).

One GPU is available, so the multi-rank case runs two processes on the
same device (IPC between processes of one device exercises the same handle
export / open / peer-store path as NVLink peers); no kernel waits on
another rank's kernel -- the ranks meet only in gloo barriers."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_06814_b200 import _native
    _native.load()


def _workload():
    from paper_1707_06814_b200.workloads import generate
    return generate(1, scale=0.1)


def _reference_k1(w):
    import torch

    from paper_1707_06814_b200 import EmbeddingParams
    from paper_1707_06814_b200.embed import embed_device_csr
    dev = torch.device("cuda", 0)
    d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
    d_off = torch.from_numpy(w.offsets).to(dev)
    emb = embed_device_csr(EmbeddingParams(128, 7), d_tok, d_off, w.d)
    return emb.values.copy(), emb.sketches(8, 7).copy()


def test_multi_destination_rows_and_offsets():
    """Two destinations, the sets computed in three row ranges: both
    destinations hold the full single-launch result."""
    import ctypes

    import torch

    from paper_1707_06814_b200 import EmbeddingParams
    from paper_1707_06814_b200._native import Context, K1Dsts
    from paper_1707_06814_b200.distributed import shard_range
    from paper_1707_06814_b200.hashing import sketch_family
    w = _workload()
    vals_ref, sk_ref = _reference_k1(w)
    ctx = Context.get()
    dev = torch.device("cuda", 0)
    d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
    d_off = torch.from_numpy(w.offsets).to(dev)
    n = w.n
    va = [torch.zeros((n, 128), dtype=torch.int32, device=dev) for _ in range(2)]
    sa = [torch.zeros((n, 8), dtype=torch.int64, device=dev) for _ in range(2)]
    efam = EmbeddingParams(128, 7).device(ctx)
    sfam = sketch_family(8, 7).device(ctx)
    stream = torch.cuda.current_stream().cuda_stream
    for r in range(3):
        lo, hi, _ = shard_range(n, r, 3)
        for fam, bufs, is_sk in ((efam, va, False), (sfam, sa, True)):
            dst = K1Dsts()
            for i, b in enumerate(bufs):
                if is_sk:
                    dst.d_sketch[i] = b.data_ptr()
                else:
                    dst.d_values[i] = b.data_ptr()
            dst.n_dsts, dst.row0 = 2, lo
            ctx.check(ctx.lib.cpsj_minhash_sketch_multi(ctx.handle, fam.handle, d_tok.data_ptr(),
                                                        d_off.data_ptr() + 8 * lo, hi - lo, w.d - 1,
                                                        ctypes.byref(dst), stream))
    torch.cuda.synchronize()
    for b in va:
        assert np.array_equal(b.cpu().numpy().view(np.uint32), vals_ref)
    for b in sa:
        assert np.array_equal(b.cpu().numpy().view(np.uint64), sk_ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_1707_06814_b200 import EmbeddingParams
    from paper_1707_06814_b200._native import Context
    from paper_1707_06814_b200.distributed import PeerArrays, embed_sharded_p2p
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = _workload()
        dev = torch.device("cuda", 0)
        d_tok = torch.from_numpy(w.tokens.view(np.int32)).to(dev)
        d_off = torch.from_numpy(w.offsets).to(dev)
        ctx = Context.get()
        peers = PeerArrays(ctx, w.n, 128, 8, rank, world)
        for _ in range(2):      # twice: the buffers are reused across steps
            vals, sk = embed_sharded_p2p(EmbeddingParams(128, 7), d_tok, d_off, w.d, (8, 7), rank, world, peers)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), values=vals.cpu().numpy().view(np.uint32),
                 sketch=sk.cpu().numpy().view(np.uint64))
        dist.barrier()
        peers.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_all_gather_two_processes(world, tmp_path):
    import torch.multiprocessing as mp
    w = _workload()
    vals_ref, sk_ref = _reference_k1(w)
    mp.spawn(_rank_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(z["values"], vals_ref)
        assert np.array_equal(z["sketch"], sk_ref)
