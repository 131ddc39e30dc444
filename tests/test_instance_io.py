"""Interchange formats either side of the scorer, CPU only.

* instance JSON (``wfsched.instance@1``, reference ``model.py:322-422``):
  files written by the reference serialiser (tests/golden/instances/, made by
  make_instance_json.py) load in the mirror, re-serialise byte-identically,
  and pack to the same SoA as the mirror's own generator output;
* binary bank (``fate.bank@1``): save -> load restores every ``fate_bank``
  array bit for bit and the index tables state packing depends on.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2605_07238_b200 import pack, scenarios
from paper_2605_07238_b200.wf import instance_io as IO
from paper_2605_07238_b200.wf import weights as MC
from paper_2605_07238_b200.wf import workloads as MB

from cases import c5_case, edge_case

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "instances")
FIXTURES = ("c1", "prefix", "override")


def _text(name):
    with open(os.path.join(GOLD, f"{name}.json")) as fh:
        return fh.read()


@pytest.mark.parametrize("name", FIXTURES)
def test_reference_instance_json_round_trips_byte_identically(name):
    text = _text(name)
    inst = IO.instance_from_json(text)
    assert IO.instance_to_json(inst) == text
    dag_text = IO.dag_to_json(inst.dag)
    assert IO.dag_to_json(IO.dag_from_json(dag_text)) == dag_text
    assert inst.dag.annotations is not None


def test_override_fixture_fields():
    inst = IO.instance_from_json(_text("override"))
    st = inst.dag.stages
    assert st["b"].base_cost_override == {"gpu0": 2.5, "gpu1": 3.25}
    assert st["c"].role is None and st["c"].model is None and st["c"].keep_cache
    assert st["a"].cache_reuse and st["a"].shared_prefix_group == "g0"
    assert inst.dag.parents("b") == ("a",) and inst.dag.children("a") == ("b", "c")
    assert inst.prefix_groups == {"g0": 2}
    assert inst.queries[1].prefix_group is None


def test_c1_fixture_equals_generated_instance_and_packs_identically():
    cfg = MC.default_config(4)
    gen = MB.lifted_instance("soykb", cfg, seed=11, batch_size=16, scale=1.0, min_groups=50)
    loaded = IO.instance_from_json(_text("c1"))
    assert IO.instance_to_json(gen) == _text("c1")
    assert loaded.dag.annotations == gen.dag.annotations
    a = pack.pack_bank([loaded], cfg.models, cfg.topology)
    b = pack.pack_bank([gen], cfg.models, cfg.topology)
    assert a.arrays.keys() == b.arrays.keys()
    for k in a.arrays:
        assert np.array_equal(a.arrays[k], b.arrays[k]), k
    assert a.scalars == b.scalars


@pytest.mark.parametrize("bad", ["wfsched.instance@2", None])
def test_unknown_schema_is_rejected(bad):
    import json

    doc = json.loads(_text("override"))
    doc["schema"] = bad
    with pytest.raises(ValueError, match="unsupported instance schema"):
        IO.instance_from_json(json.dumps(doc))
    dag = json.loads(_text("override"))["dag"]
    dag["schema"] = "wfsched.dag@0"
    with pytest.raises(ValueError, match="unsupported dag schema"):
        IO.dag_from_json(json.dumps(dag))


@pytest.mark.parametrize("make", [lambda: edge_case(), lambda: c5_case(n_inst=3)])
def test_bank_file_round_trip(tmp_path, make):
    case = make()
    path = tmp_path / "bank.npz"
    pack.save_bank(case.bank, path)
    got = pack.load_bank(path)
    src = case.bank
    assert got.arrays.keys() == src.arrays.keys()
    for k, v in src.arrays.items():
        assert got.arrays[k].dtype == v.dtype and np.array_equal(got.arrays[k], v), k
    assert got.scalars == src.scalars
    assert got.device_ids == src.device_ids and got.model_index == src.model_index
    assert got.group_index == src.group_index and got.n_models == src.n_models
    assert got.stage_ids == [list(s) for s in src.stage_ids]
    # a state packs the same against the reloaded bank (index tables intact)
    n_inst = len(src.stage_ids)
    scen = []
    for i in range(n_inst):
        inst = src.instances[i]
        cfg = scenarios.config_c5() if case.name.startswith("c5") else None
        if cfg is None:
            break
        scen.append((i, scenarios.build_scenario(inst, cfg, i)))
    if scen:
        s_src = pack.pack_states(src, scen)
        s_got = pack.pack_states(got, scen)
        for k in s_src.arrays:
            assert np.array_equal(s_src.arrays[k], s_got.arrays[k]), k


def test_bank_file_rejects_foreign_format(tmp_path):
    path = tmp_path / "x.npz"
    np.savez(path, meta=np.frombuffer(b'{"format": "other"}', np.uint8),
             ids=np.zeros(0, np.uint8))
    with pytest.raises(ValueError, match="unsupported bank format"):
        pack.load_bank(path)
