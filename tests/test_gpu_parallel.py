"""parallel.predict_shard on the GPU: every rank's contiguous shard scored by K1
reassembles the single-process batch bit for bit (examples are independent,
M:321-397), for world sizes 1-4 and an uneven batch."""

import numpy as np
import pytest
import torch

from oracle import fieldwise_oracle as fo
from paper_2407_10115_b200 import configs, synth
from paper_2407_10115_b200.model import ModelConfig, WeightStore, predict_batch
from paper_2407_10115_b200.parallel import predict_shard, shard_range

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_predict_shard_reassembles_the_full_batch(world):
    wl = configs.CFG2
    ost = fo.random_store(wl.n_fields, wl.k, wl.hidden, 12, seed=31)
    cfg = ModelConfig(n_fields=wl.n_fields, k=wl.k, hidden_sizes=wl.hidden, hash_bits=12)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, with_optimizer=False)
    n = 5003
    idx, val = synth.make_examples(wl, n, seed=32, hash_bits=12, device=DEV)
    full = predict_batch(idx, val, st).cpu().numpy()
    got = np.empty(n, np.float32)
    for r in range(world):
        sh = shard_range(n, world, r)
        got[sh.start:sh.stop] = predict_shard(idx, val, st, sh).cpu().numpy()
    assert np.array_equal(got, full)
