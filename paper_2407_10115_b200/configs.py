"""The five BASELINE.json workloads as concrete, seeded synthetic recipes.

SURVEY.md section 8(d) is the source of every number here.  The paper's
datasets (Criteo / Avazu / KDD2012) are not in the container;
these seeded synthetic streams stand in for them with the structural traits
that matter to this path: hashed categorical fields with value 1.0, a few
positive numeric fields, and Zipf-skewed feature frequencies.
"""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Workload:
    name: str
    n_fields: int
    k: int
    hash_bits: int
    hidden: tuple
    max_per_field: int  # M: padded feature slots per field
    n_examples: int
    dist: str  # "uniform" | "zipf"
    zipf_alpha: float = 1.1
    numeric_fields: tuple = ()  # fields with LogNormal(0,1) values
    weight_scale: float = 0.05
    weight_dtype: str = "f32"  # f32 | bf16 | u16
    label_p: float = 0.3
    data_seed: int = 2000
    weight_seed: int = 1000
    # cfg3 (training)
    lr: float = 0.1
    power_t: float = 0.5
    # cfg4 (serving)
    n_requests: int = 0
    n_candidates: int = 0
    ctx_fields: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def n_pairs(self):
        return self.n_fields * (self.n_fields - 1) // 2


CFG1 = Workload("cfg1_ffm_lr", 8, 4, 18, (), 1, 65_536, "uniform", weight_scale=0.1,
                data_seed=2001, weight_seed=1001)
CFG2 = Workload("cfg2_deepffm_fwd", 24, 8, 24, (64, 32), 3, 1_048_576, "zipf", 1.1,
                numeric_fields=(20, 21, 22, 23), data_seed=2002, weight_seed=1002)
CFG3 = Workload("cfg3_adagrad", 24, 8, 24, (64, 32), 3, 10_000_000, "zipf", 1.1,
                numeric_fields=(20, 21, 22, 23), data_seed=2003, weight_seed=1003)
CFG4 = Workload("cfg4_ctx_cache_u16", 24, 8, 24, (64, 32), 1, 1_000_000, "zipf", 1.1,
                weight_dtype="u16", data_seed=2004, weight_seed=1004,
                n_requests=2000, n_candidates=500, ctx_fields=16)
CFG5 = Workload("cfg5_large_bf16", 40, 16, 25, (256, 128), 1, 8_388_608, "zipf", 1.05,
                weight_dtype="bf16", data_seed=2005, weight_seed=1005)

WORKLOADS = {w.name: w for w in (CFG1, CFG2, CFG3, CFG4, CFG5)}
BY_ID = {1: CFG1, 2: CFG2, 3: CFG3, 4: CFG4, 5: CFG5}
