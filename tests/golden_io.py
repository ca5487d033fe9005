"""Load the reference-generated golden fixtures (see tests/golden/make_golden.py)."""

import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=True)


def n_weights(F, k, hidden, bits):
    nb = 1 << bits
    total = nb + 1 + nb * F * k
    if len(hidden):
        dims = [1 + F * (F - 1) // 2, *[int(h) for h in hidden], 1]
        total += sum(i * o + o for i, o in zip(dims[:-1], dims[1:]))
    return total


def seeded_flat(F, k, hidden, bits, seed, scale, bf16=False):
    """Regenerate the fixture's weights (default_rng(seed) normal * scale, f32)."""
    n = n_weights(F, k, hidden, bits)
    flat = (np.random.default_rng(int(seed)).standard_normal(n) * float(scale)).astype(np.float32)
    if bf16:
        import torch
        flat = torch.from_numpy(flat).to(torch.bfloat16).to(torch.float32).numpy()
    return flat


def fixture_flat(g):
    F, k, bits = int(g["F"]), int(g["k"]), int(g["bits"])
    hidden = tuple(int(h) for h in g["hidden"])
    bf16 = bool(g["bf16"]) if "bf16" in g.files else False
    flat = seeded_flat(F, k, hidden, bits, g["w_seed"], g["scale"], bf16)
    if "flat_sha" in g.files:
        assert hashlib.sha256(flat.tobytes()).hexdigest() == str(g["flat_sha"]), \
            "weight regeneration drifted from the golden fixture"
    return F, k, hidden, bits, flat
