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
  ``cli.py:30``; reference signature ``make_policy(name, beam=None,
  solver_budget_s=0.25)``, ``policies.py:504``) -- "fate" returns
  :class:`~.planner.FateGpuPolicy`, a subclass of the caller's FatePolicy
  whose S matrix and work-conserving timings also come from the GPU;
* with ``mirror=`` a :class:`~.mirror.MirrorScorer`: ``wfsched.executor``'s
  ``ExecutionState`` name is wrapped so the live state of every run is
  attached to the device-resident mirror (its transitions, ``state.py:130-184``,
  become device events), and -- if the mirror provides the frontier --
  ``wfsched.executor.ready_set`` answers from the GPU ready set
  (``model.py:306-319``, called at ``executor.py:192``);
* with ``durations=True``: ``wfsched.executor.CostModel`` (constructed by
  ``run`` at ``executor.py:168``) becomes :class:`~.durations.GpuCostModel`,
  so the executor's issue-time ``realized_duration`` (``executor.py:231-233``)
  is priced on the GPU.
CSV ``method`` stays "fate", so the reference's tables remain comparable.
"""

from __future__ import annotations

import importlib

_saved: dict = {}
_bound: dict = {}


def _set(mod, name: str, value) -> None:
    if (mod, name) not in _saved:
        _saved[(mod, name)] = getattr(mod, name)
    setattr(mod, name, value)


def install(scorer=None, policy_factory: bool = True, mirror=None,
            durations: bool = False) -> None:
    """Reroute the reference's FATE cost matrix (and, by default, the whole
    FATE policy) through the GPU scorer.  A second call with the same
    arguments is a no-op; with different ones it raises -- call
    :func:`uninstall` first."""
    from .planner import FateGpuPolicy, build_problem

    chosen = mirror if (mirror is not None and scorer is None) else scorer
    args = {"scorer": chosen, "policy_factory": policy_factory, "mirror": mirror,
            "durations": durations}
    if _saved:
        if all(_bound.get(k) is v for k, v in args.items()):
            return
        raise RuntimeError("compat.install() is already active with other arguments; "
                           "call compat.uninstall() first")
    pol = importlib.import_module("wfsched.policies")
    ex = importlib.import_module("wfsched.executor")

    def gpu_build_problem(frontier, state, cost_model, dag):
        return build_problem(frontier, state, cost_model, dag, scorer=chosen)

    _set(pol, "build_problem", gpu_build_problem)
    if policy_factory:
        original = pol.make_policy

        def make_policy(name: str, beam=None, solver_budget_s: float = 0.25):
            if name == "fate":
                return FateGpuPolicy(solver_budget_s=solver_budget_s, scorer=chosen)
            return original(name, beam=beam, solver_budget_s=solver_budget_s)

        for modname in ("wfsched.policies", "wfsched.harness", "wfsched.cli"):
            mod = importlib.import_module(modname)
            if hasattr(mod, "make_policy"):
                _set(mod, "make_policy", make_policy)
    if durations:
        from . import durations as dur

        dur.set_source(mirror if mirror is not None else scorer)
        _set(ex, "CostModel", dur.GpuCostModel)
    if mirror is not None:
        real_state = ex.ExecutionState
        real_ready = ex.ready_set

        class _LiveState:
            """``ExecutionState`` as the executor names it: ``initial`` builds
            the real state and attaches it to the device mirror."""

            @staticmethod
            def initial(instance, device_ids, record_trace: bool = False):
                st = real_state.initial(instance, device_ids, record_trace=record_trace)
                mirror.attach_live(st)
                return st

        def ready_set(dag, completed, running=frozenset(), committed=frozenset()):
            if getattr(mirror, "provides_frontier", False) and mirror.follows(dag):
                return mirror.frontier()
            return real_ready(dag, completed, running, committed)

        _set(ex, "ExecutionState", _LiveState)
        _set(ex, "ready_set", ready_set)
    _bound.update(args)


def uninstall() -> None:
    for (mod, name), value in _saved.items():
        setattr(mod, name, value)
    if _bound.get("durations"):
        from . import durations as dur

        dur.set_source(None)
    _saved.clear()
    _bound.clear()
