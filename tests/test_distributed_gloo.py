"""Repetition sharding over 2 ranks (gloo, CPU): the gathered, deduplicated
pair set and the all-reduced counters equal the single-process join.

The per-rank local join is injected (the C oracle restricted to the rank's
repetition seeds) because this container has no GPU; the exchange logic
under test -- rep assignment, variable-size all-gather, sort + unique,
sum/max reductions -- is the product code in paper_1707_06814_b200.distributed.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _workload():
    from paper_1707_06814_b200.workloads import generate
    return generate(1, scale=0.05)


def _oracle_local(w, values, sk):
    from paper_1707_06814_b200.core import Counters
    from paper_1707_06814_b200.cpsjoin import JoinArrays, make_plan

    def local(emb, params, rep_indices):
        plan = make_plan(params, values.shape[1])
        seeds = plan.rep_seeds[rep_indices]
        # run the oracle tree by tree with explicit seeds
        keys, sims, ev = [], [], []
        c = [0, 0, 0, 0, 0]
        for s in seeds:
            out = _oracle_with_seed(w, values, sk, params, int(s))
            keys.append(out.keys)
            sims.append(out.sims)
            ev.append(out.cap_events)
            c[0] += out.pre_candidates
            c[1] += out.candidates
            c[2] += out.results
            c[3] = max(c[3], out.max_depth)
            c[4] = max(c[4], out.peak_live_members)
        k = np.concatenate(keys) if keys else np.zeros(0, np.uint64)
        s_ = np.concatenate(sims) if sims else np.zeros(0)
        k, first = np.unique(k, return_index=True)
        a = (k >> np.uint64(32)).astype(np.int64)
        b = (k & np.uint64(0xFFFFFFFF)).astype(np.int64)
        return JoinArrays(a, b, s_[first], Counters(*c), np.concatenate(ev) if ev else np.zeros(0, np.int64), {})
    return local


def _oracle_with_seed(w, values, sk, params, seed):
    import ctypes
    L = O.lib()
    tok, off = O._csr(w.tokens, w.offsets)
    sizes = np.ascontiguousarray(w.sizes, dtype=np.int64)
    seeds = np.array([seed], dtype=np.uint64)
    kp, sp, cp = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    nk, nc = ctypes.c_int64(), ctypes.c_int64()
    counters = np.zeros(5, dtype=np.int64)
    ks = O.kstar(params.lambda_, params.delta, 64 * params.ell)
    L.orc_self_join(O._p(tok), O._p(off), O._p(sizes), len(off) - 1, O._p(values), values.shape[1], O._p(sk),
                    sk.shape[1], params.lambda_, params.epsilon, params.limit, ks, params.depth_cap, O._p(seeds), 1, 1,
                    ctypes.byref(kp), ctypes.byref(sp), ctypes.byref(nk), O._p(counters), ctypes.byref(cp),
                    ctypes.byref(nc))
    return O.JoinOut(O._take(kp, nk.value, np.uint64), O._take(sp, nk.value, np.float64), *counters.tolist(),
                     O._take(cp, nc.value, np.int64), 0)


def _rank_main(rank, world, port, q):
    import torch.distributed as dist

    from paper_1707_06814_b200.cpsjoin import CPSJoinParams
    from paper_1707_06814_b200.distributed import shard_reps
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = _workload()
        values = O.minhash(w.tokens, w.offsets, O.embedding_tables(128, 7), 1)
        mh, bt = O.sketch_tables(8, 7)
        sk = O.sketch(w.tokens, w.offsets, mh, bt, 1)
        params = CPSJoinParams(lambda_=0.5, seed=7, repetitions=5)
        res = shard_reps(None, params, rank, world, local_join=_oracle_local(w, values, sk))
        c = res.counters
        q.put((rank, res.a.tolist(), res.b.tolist(), res.similarity.tolist(),
               [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members]))
    finally:
        dist.destroy_process_group()


def test_two_rank_rep_sharding_equals_single_process():
    w = _workload()
    ref = O.full_pipeline(w.tokens, w.offsets, w.sizes, lam=0.5, emb_seed=7, seed=7, repetitions=5, threads=1)[2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, a, b, s, c in outs:
        assert a == ref.a.tolist() and b == ref.b.tolist()
        assert s == ref.sims.tolist()
        assert c == [ref.pre_candidates, ref.candidates, ref.results, ref.max_depth, ref.peak_live_members]


def _oracle_k1(w):
    """CPU stand-in for the K1 launch of one rank (test only)."""
    import torch

    def k1(eparams, sketch, d_tok, d_off, d, lo, hi, vals_out, sk_out):
        off = w.offsets[lo:hi + 1]
        tok = w.tokens[off[0]:off[-1]]
        rel = off - off[0]
        vals_out[:hi - lo] = torch.from_numpy(O.minhash(tok, rel, eparams.tables, 1).view(np.int32))
        if sketch is not None:
            mh, bt = O.sketch_tables(*sketch)
            sk_out[:hi - lo] = torch.from_numpy(O.sketch(tok, rel, mh, bt, 1).view(np.int64))
    return k1


def _shard_main(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1707_06814_b200.distributed import embed_sharded
    from paper_1707_06814_b200.embed import EmbeddingParams
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = _workload()
        ep = EmbeddingParams(t=32, seed=7)
        d_tok = torch.from_numpy(w.tokens.view(np.int32))
        d_off = torch.from_numpy(w.offsets)
        vals, sk = embed_sharded(ep, d_tok, d_off, w.d, (2, 7), rank, world, local_k1=_oracle_k1(w))
        q.put((rank, vals.numpy().view(np.uint32).tolist(), sk.numpy().view(np.uint64).tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_set_sharded_embedding_all_gathers_full_matrices(world):
    w = _workload()
    ref_vals = O.minhash(w.tokens, w.offsets, O.embedding_tables(32, 7), 1)
    mh, bt = O.sketch_tables(2, 7)
    ref_sk = O.sketch(w.tokens, w.offsets, mh, bt, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, vals, sk in outs:
        assert np.array_equal(np.array(vals, dtype=np.uint32), ref_vals)
        assert np.array_equal(np.array(sk, dtype=np.uint64), ref_sk)


def test_shard_ranges_cover_every_set_once():
    from paper_1707_06814_b200.distributed import shard_range
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            got = [shard_range(n, r, world)[:2] for r in range(world)]
            covered = [i for lo, hi in got for i in range(lo, hi)]
            assert covered == list(range(n))


def test_merge_results_is_order_independent():
    from paper_1707_06814_b200.distributed import merge_results
    rng = np.random.default_rng(0)
    keys = rng.integers(0, 1000, size=300).astype(np.uint64)
    sims = keys.astype(np.float64) / 1000.0  # equal keys carry equal sims
    k1, s1 = merge_results(keys, sims)
    perm = rng.permutation(len(keys))
    k2, s2 = merge_results(keys[perm], sims[perm])
    assert np.array_equal(k1, k2) and np.array_equal(s1, s2)
    assert np.all(np.diff(k1.astype(np.int64)) > 0)


def _frontier_main(rank, world, depth, port, q):
    """One rank of shard_frontier (the bench's N > 1 default) with the C
    oracle's frontier mode as the injected local join."""
    import torch.distributed as dist

    from paper_1707_06814_b200.core import Counters
    from paper_1707_06814_b200.cpsjoin import CPSJoinParams, JoinArrays
    from paper_1707_06814_b200.distributed import shard_frontier
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = _workload()
        values = O.minhash(w.tokens, w.offsets, O.embedding_tables(128, 7), 1)
        mh, bt = O.sketch_tables(8, 7)
        sk = O.sketch(w.tokens, w.offsets, mh, bt, 1)
        params = CPSJoinParams(lambda_=0.5, seed=7, repetitions=3, limit=40)

        def local(emb, p, frontier):
            out = O.self_join(w.tokens, w.offsets, w.sizes, values, sk, p.lambda_, epsilon=p.epsilon, limit=p.limit,
                              delta=p.delta, repetitions=p.repetitions, seed=p.seed, depth_cap=p.depth_cap,
                              threads=1, frontier=frontier)
            return JoinArrays(out.a, out.b, out.sims, Counters(out.pre_candidates, out.candidates, out.results,
                                                               out.max_depth, out.peak_live_members),
                              out.cap_events, {})

        res = shard_frontier(None, params, rank, world, depth=depth, local_join=local)
        c = res.counters
        q.put((rank, res.a.tolist(), res.b.tolist(), res.similarity.tolist(),
               [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members],
               len(res.depth_cap_sizes)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,depth", [(2, 1), (3, 2)])
def test_frontier_sharding_over_ranks_equals_single_process(world, depth):
    """shard_frontier across `world` gloo processes (frontier cut, variable
    all-gather of pairs, sort + unique, counter sum/max) equals the
    unsharded join on every rank."""
    w = _workload()
    values = O.minhash(w.tokens, w.offsets, O.embedding_tables(128, 7), 1)
    mh, bt = O.sketch_tables(8, 7)
    sk = O.sketch(w.tokens, w.offsets, mh, bt, 1)
    ref = O.self_join(w.tokens, w.offsets, w.sizes, values, sk, 0.5, repetitions=3, seed=7, limit=40, threads=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_frontier_main, args=(r, world, depth, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, a, b, s, c, ncap in outs:
        assert a == ref.a.tolist() and b == ref.b.tolist()
        assert s == ref.sims.tolist()
        assert c == [ref.pre_candidates, ref.candidates, ref.results, ref.max_depth, ref.peak_live_members]
        assert ncap == len(ref.cap_events)
