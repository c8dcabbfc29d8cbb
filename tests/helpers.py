"""Shared test helpers: config builders mirroring the reference tests'
make_config (proj/tests/test_bubblefill.cpp:20-29, acceptance.cpp:53-61) and
canonical dumps of product schedules."""
from paper_2211_14133_b200 import schedule as S


class SplitMix64:
    """proj/src/kfac/kfac.cpp:228-238 (the reference tests' seeded RNG)."""

    def __init__(self, seed: int):
        self.state = seed & 0xFFFFFFFFFFFFFFFF

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53

    def symmetric(self) -> float:
        return 2.0 * self.uniform() - 1.0


def make_config(method, depth, n_micro, layers=1, replicas=0):
    return S.PipelineConfig(method=S.Method(method), stages=depth, micro_batches=n_micro,
                            layers_per_stage=layers,
                            replicas=replicas if replicas > 0 else
                            (2 if S.Method(method) == S.Method.Chimera else 1))


def hand_costs():
    return S.CostTable(t_f=1.0, t_b=1.0, t_curv=0.5, t_inv=1.0, t_prec=0.25)


def item_tuple(w):
    return (w.device, int(w.kind), w.stage, -1 if w.micro_batch is None else w.micro_batch,
            -1 if w.layer is None else w.layer, -1 if w.factor is None else int(w.factor),
            w.start, w.duration, w.step)


def items_of(schedule):
    return [item_tuple(w) for line in schedule.timelines for w in line]


def canonical(items):
    return sorted(items, key=lambda t: (t[0], t[6], t[1], t[2], t[3], t[4], t[5], t[8], t[7]))


def acceptance_table(rng: SplitMix64):
    """One seeded cost table exactly as proj/tests/acceptance.cpp:205-230 draws it."""
    method = [0, 1, 2][rng.next() % 3]
    depth = 2 + 2 * (rng.next() % 2) if method == 2 else 2 + rng.next() % 3
    n = depth * (1 + rng.next() % 2)
    layers = 1 + rng.next() % 3
    cfg = make_config(method, depth, n, layers)
    if rng.next() % 4 == 0:
        cfg.replicas *= 2
    inv_par = rng.next() % 2 == 0 and cfg.replicas > 1
    costs = S.CostTable(t_f=1.0)
    costs.t_b = 0.5 + 1.5 * rng.uniform()
    costs.t_curv = 2.0 * rng.uniform() * costs.t_f
    costs.t_inv = 2.0 * rng.uniform() * costs.t_f
    costs.t_prec = 2.0 * rng.uniform() * costs.t_f
    return cfg, costs, inv_par


def soundness_table(rng: SplitMix64):
    """proj/tests/test_bubblefill.cpp:320-334 (seed 271828)."""
    method = [0, 1, 2][rng.next() % 3]
    depth = 2 + 2 * (rng.next() % 2) if method == 2 else 2 + rng.next() % 3
    n = depth * (1 + rng.next() % 2)
    layers = 1 + rng.next() % 3
    cfg = make_config(method, depth, n, layers)
    costs = S.CostTable(t_f=1.0)
    costs.t_b = 0.5 + 1.5 * rng.uniform()
    costs.t_curv = 2.0 * rng.uniform() * costs.t_f
    costs.t_inv = 2.0 * rng.uniform() * costs.t_f
    costs.t_prec = 2.0 * rng.uniform() * costs.t_f
    return cfg, costs


def bert_configs():
    """BASELINE.json configs 2-4 with B200-scaled costs."""
    t_f = 0.394
    base_gpipe = (S.PipelineConfig(method=S.Method.GPipe, stages=4, micro_batches=4,
                                   micro_batch_size=32, replicas=1, layers_per_stage=3),
                  S.CostTable(t_f=0.25, t_b=0.5, t_curv=0.05, t_inv=3 * 0.27, t_prec=0.08,
                              m_theta=85_000_000, m_curv=170_000_000))
    chimera = (S.PipelineConfig(method=S.Method.Chimera, stages=8, micro_batches=8,
                                micro_batch_size=32, replicas=2, layers_per_stage=3),
               S.CostTable(t_f=t_f, t_b=2 * t_f, t_curv=0.108, t_inv=3 * 74.1 / 200.0,
                           t_prec=2 * 3 * 103.0 / 700.0))
    chimera_nv = (S.PipelineConfig(method=S.Method.Chimera, stages=8, micro_batches=8,
                                   micro_batch_size=32, replicas=2, layers_per_stage=3),
                  S.CostTable(t_f=t_f, t_b=2 * t_f, t_curv=0.108, t_inv=3 * 74.1 / 200.0,
                              t_prec=2 * 3 * 103.0 / 700.0, m_theta=151_000_000,
                              m_curv=528_000_000, comm_alpha=0.01, comm_beta=7e8))
    onef1b = (S.PipelineConfig(method=S.Method.OneF1B, stages=4, micro_batches=4,
                               micro_batch_size=32, replicas=2, layers_per_stage=6),
              S.CostTable(t_f=2 * t_f, t_b=4 * t_f, t_curv=0.108, t_inv=6 * 74.1 / 200.0,
                          t_prec=6 * 103.0 / 700.0, m_theta=302_000_000, m_curv=1_056_000_000,
                          comm_alpha=0.01, comm_beta=7e8))
    return {"bert_base_gpipe_d4n4": base_gpipe, "bert_large_chimera_d8n8": chimera,
            "bert_large_chimera_d8n8_nvlink": chimera_nv, "bert_large_1f1b_d4n4w2": onef1b}
