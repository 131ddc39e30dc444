"""Walk workload of the C4 sweep: per step, how many (item,
horizon level) pairs the scoring kernel walks and how many op-list entries
those walks hold, from the packed bank and scenario states alone (CPU).

A level l of item (scenario s, stage v) is walked iff the lowest window
parent of (v, l) is at or below the scenario's highest located level (the
kernel's rule, fate_score_v6.cuh).  Its op template has, per descendant x of
the bucket, a model op (x has a model), a prefix op (x shares v's prefix
group) and one entry per parent edge of x other than v; the compaction keeps
model/prefix ops and the edges whose parent is located.

    python tools/c4_walk_stats.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_07238_b200 import runtime  # noqa: E402


def main():
    cfg, bank, states, work = bench.build_c4("sweep")
    LV = max(cfg.weights.effective_horizon() - 1, 0)
    ptr, idx = runtime.build_windows(bank, LV)
    wmin = runtime.window_parent_min_level(bank, LV)
    a = bank.arrays
    par_ptr, par_idx = a["par_ptr"], a["par_idx"]
    model, group = a["st_model"], a["st_group"]
    V = bank.n_stages
    n_scen = states.n_scenarios
    st = states.arrays
    done = st["scen_done_level"]
    loc = st["loc"].reshape(n_scen, V)
    n_items = n_scen * V
    # per (v, l): template length, and the edges (parent ids) of its bucket
    tmpl_len = np.zeros(V * LV, dtype=np.int64)
    edges = []
    for vl in range(V * LV):
        v = vl // LV
        xs = idx[ptr[vl]:ptr[vl + 1]]
        n = int((model[xs] != -1).sum()) + int(((group[xs] != -1) & (group[xs] == group[v])).sum())
        ps = np.concatenate([par_idx[par_ptr[x]:par_ptr[x + 1]] for x in xs]) if len(xs) else \
            np.zeros(0, np.int32)
        ps = ps[ps != v]
        tmpl_len[vl] = n + len(ps)
        edges.append((n, ps))
    walked = tmpl = kept = 0
    for s in range(n_scen):
        wm = wmin[: V * LV] <= done[s]
        nonempty = (ptr[1:] - ptr[:-1]) > 0
        sel = np.nonzero(wm & nonempty)[0]
        walked += len(sel)
        tmpl += int(tmpl_len[sel].sum())
        for vl in sel:
            n, ps = edges[vl]
            kept += n + int((loc[s, ps] >= 0).sum())
    print(json.dumps({"workload": "c4_sweep", "items": n_items, "levels": LV,
                      "item_levels": n_items * LV, "walked_item_levels": walked,
                      "template_entries_walked": tmpl, "entries_kept": kept,
                      "entries_per_item": tmpl / n_items,
                      "entries_per_walked_level": tmpl / max(walked, 1)}))


if __name__ == "__main__":
    main()
