"""N>1 inference sharding on CPU with the gloo backend, world size 2.

The scoring function here is the oracle (CPU); on the GPU box each rank calls
K1 on its slice instead (bench.py --gpus N).  What is tested is the sharding
logic itself: disjoint balanced cover, replicated-table agreement without data
movement, and that the ranks' slices reassemble the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_10115_b200.parallel import shard_range, table_digest


def test_shard_range_properties():
    for n in (0, 1, 7, 1000, 8_388_608):
        for world in (1, 2, 3, 4, 8):
            shards = [shard_range(n, world, r) for r in range(world)]
            assert shards[0].start == 0 and shards[-1].stop == n
            for a, b in zip(shards, shards[1:]):
                assert a.stop == b.start
            sizes = [s.size for s in shards]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import fieldwise_oracle as fo
    from paper_2407_10115_b200 import configs, synth
    wl = configs.CFG2
    # replicated tables: every rank generates them from the same seed
    st = fo.random_store(wl.n_fields, wl.k, wl.hidden, 10, seed=wl.weight_seed)
    dig = table_digest(st.lr, st.ffm)
    digs = [None] * world
    dist.all_gather_object(digs, dig)
    # the full batch is a deterministic function of the seed; each rank scores
    # only its shard, no data-path collective
    n = 203
    idx, val = synth.make_examples(wl, n, seed=11, hash_bits=10)
    sh = shard_range(n, world, rank)
    _, p = fo.forward_batch(idx.numpy()[sh.start:sh.stop], val.numpy()[sh.start:sh.stop], st)
    parts = [None] * world
    dist.all_gather_object(parts, (sh.start, sh.stop, p))  # test-only reassembly
    if rank == 0:
        q.put((digs, parts))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_inference_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    digs, parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(set(digs)) == 1  # tables identical on every rank
    from oracle import fieldwise_oracle as fo
    from paper_2407_10115_b200 import configs, synth
    wl = configs.CFG2
    st = fo.random_store(wl.n_fields, wl.k, wl.hidden, 10, seed=wl.weight_seed)
    idx, val = synth.make_examples(wl, 203, seed=11, hash_bits=10)
    _, full = fo.forward_batch(idx.numpy(), val.numpy(), st)
    got = np.empty(203)
    covered = 0
    for a, b, p in parts:
        got[a:b] = p
        covered += b - a
    assert covered == 203
    np.testing.assert_array_equal(got, full)


def _bcast_worker(rank, world, port, q):
    """parallel.broadcast_store itself: rank 0 holds the trained blocks (f32 with
    accumulators, and a u16 store with its host-side headers), rank 1 starts empty."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_10115_b200.model import ModelConfig, WeightStore
    from paper_2407_10115_b200.parallel import broadcast_store
    cfg = ModelConfig(n_fields=4, k=2, hidden_sizes=(8,), hash_bits=10)
    st = WeightStore(cfg, "cpu")
    sq = WeightStore(cfg, "cpu", "u16", with_optimizer=False)
    if rank == 0:
        g = torch.Generator().manual_seed(1)
        for _, t in st.blocks(True):
            t.copy_(torch.randn(t.shape, generator=g))
        for _, t in sq.blocks(False):
            if t.dtype == torch.uint16:
                t.copy_(torch.randint(0, 65536, t.shape, generator=g).to(torch.uint16))
            else:
                t.copy_(torch.randn(t.shape, generator=g))
        sq.q_headers = {"lr": (-0.5, 1e-5), "ffm": (-0.25, 2e-6)}
    broadcast_store(st)
    broadcast_store(sq)
    digs = [table_digest(*[t.numpy().view(np.uint8) if t.dtype != torch.uint16
                           else t.view(torch.int16).numpy() for _, t in x.blocks(x.has_optimizer)])
            for x in (st, sq)]
    out = [None] * world
    dist.all_gather_object(out, (digs, sq.q_headers, st.version))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_broadcast_store_replicates_every_block():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (d0, h0, v0), (d1, h1, v1) = out
    assert d0 == d1  # f32 + accumulators and u16 tables byte-identical on both ranks
    assert h0 == h1 == {"lr": (-0.5, 1e-5), "ffm": (-0.25, 2e-6)}
    assert v0 == v1 == 1  # the broadcast marks the store mutated
