"""Install the GPU scorer into an existing ``wfsched`` (the reference package).

    import wfsched
    from paper_2605_07238_b200 import compat
    compat.install()          # "fate" now plans with the sm_100a scorer
    ...                       # wfsched.cli / harness / executor unchanged
    compat.uninstall()

Patch points (SURVEY.md §8(b) "Integration points"):
* ``wfsched.policies.build_problem`` -- FatePolicy binds it at import
  (``policies.py:19``), so replacing the module global reroutes the cost
  matrix of any FatePolicy instance (``policies.py:62``);
* ``make_policy`` in ``wfsched.policies`` / ``wfsched.harness`` /
  ``wfsched.cli`` (the closed factory imported by name, ``harness.py:47``,
  ``cli.py:30``) -- "fate" returns :class:`FateGpuPolicy`, which also takes the
  horizon-0 S matrix and the work-conserving completion matrix from the GPU.
CSV ``method`` stays "fate", so the reference's tables remain comparable.
"""

from __future__ import annotations

import importlib

from .planner import FateGpuPolicy, GpuScorer, build_problem

_saved: dict = {}


def install(scorer: GpuScorer | None = None, policy_factory: bool = True) -> None:
    """Reroute the reference's FATE cost matrix (and, by default, the whole
    FATE policy) through the GPU scorer."""
    if _saved:
        return
    pol = importlib.import_module("wfsched.policies")
    chosen = scorer

    def gpu_build_problem(frontier, state, cost_model, dag):
        return build_problem(frontier, state, cost_model, dag, scorer=chosen)

    _saved[(pol, "build_problem")] = pol.build_problem
    pol.build_problem = gpu_build_problem
    if policy_factory:
        original = pol.make_policy

        def make_policy(name: str):
            if name == "fate":
                return FateGpuPolicy(scorer=chosen) if chosen is not None else FateGpuPolicy()
            return original(name)

        for modname in ("wfsched.policies", "wfsched.harness", "wfsched.cli"):
            mod = importlib.import_module(modname)
            if hasattr(mod, "make_policy"):
                _saved[(mod, "make_policy")] = mod.make_policy
                mod.make_policy = make_policy


def uninstall() -> None:
    for (mod, name), value in _saved.items():
        setattr(mod, name, value)
    _saved.clear()
