"""Oracle-backed scorer with the GpuScorer interface (test infrastructure).

Lets the CPU test suite drive the reference executor and the GPU policy's
host side with the C oracle, to validate the host side of the drop-in without a GPU.  Never used
by the product.
"""

from __future__ import annotations

import oracle
from paper_2605_07238_b200 import pack
from paper_2605_07238_b200.planner import WaveScores


class OracleScorer:
    def __init__(self):
        self._cache = {}

    def _bank(self, instance, cost_model):
        key = (id(instance), id(cost_model.models), id(cost_model.topo))
        hit = self._cache.get(key)
        if hit is None or hit[0] is not instance:
            hit = (instance, pack.pack_bank([instance], cost_model.models, cost_model.topo))
            self._cache = {key: hit}
        return hit[1]

    def score_wave(self, frontier, state, cost_model, dag=None) -> WaveScores:
        bank = self._bank(state.instance, cost_model)
        wrec = pack.weights_record(cost_model.weights)
        sids = sorted(frontier)
        states = pack.pack_states(bank, [(0, state)])
        work = pack.make_work(bank, [(0, bank.global_index(0, s)) for s in sids],
                              cost_model.weights.ablation.no_shard)
        res = oracle.score(bank, wrec, states, work, n_threads=1)
        D = bank.scalars["n_devices"]
        n = len(sids)
        return WaveScores(
            stage_ids=sids, bounds=[int(b) for b in work.bounds], device_ids=bank.device_ids,
            elig=[int(bank.arrays["st_elig"][g]) for g in work.stage], psi=res["psi"],
            psi_off=work.psi_off, sched=res["sched"].reshape(n, D),
            completion=res["completion"].reshape(n, D), tail=res["tail"].reshape(n, D),
            timing=res["timing"].reshape(n, D, 3))
