"""Score weights, ablation switches and the shipped default catalogs.

Mirror of the scorer-facing part of ``wfsched.config`` (reference
``pkg/src/wfsched/config.py:24-182``).  ``ScoreWeights`` and
``AblationFlags`` are the kernel's constant bank (packed into the POD
``fate_weights`` struct, ``include/fate.h``).  YAML I/O is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

from .dagmodel import DeviceSpec, DeviceTopology, ModelProfile, StageRole

DEFAULT_SEED = 20260423

# alias: (memory_gb, prefill_coeff, decode_coeff, switch_penalty)   -- config.py:24-30
_MODEL_ROWS = (
    ("qwen-7b", 15.0, 0.8, 0.0010, 12.0),
    ("deepseek-7b", 15.0, 1.0, 0.0013, 15.0),
    ("llama-8b", 17.0, 0.9, 0.0011, 18.0),
)

# kind: complexity, prefill, decode, max_tok, out_tok, comm, keep, reuse, shard -- config.py:35-48
_ROLE_ROWS = {
    "prompt_prep": (0.6, 0.8, 0.5, 2048, 256, 1.0, True, True, True),
    "retrieval": (0.8, 1.2, 0.4, 4096, 512, 2.0, True, True, True),
    "routing": (0.5, 0.6, 0.3, 1024, 128, 0.5, False, True, True),
    "decomposition": (1.0, 1.0, 0.8, 2048, 384, 1.5, True, True, True),
    "worker": (1.4, 1.0, 1.0, 4096, 512, 1.0, False, True, True),
    "merge": (1.1, 1.3, 0.7, 3072, 512, 3.0, False, False, False),
    "aggregation": (1.2, 1.4, 0.8, 3072, 640, 3.0, False, False, False),
    "summarization": (1.0, 1.1, 0.9, 4096, 384, 1.5, True, True, True),
    "validation": (0.7, 0.9, 0.5, 2048, 192, 1.0, False, True, True),
    "verification": (0.8, 1.0, 0.6, 2048, 192, 1.0, False, True, True),
    "final_synthesis": (1.2, 1.2, 1.1, 4096, 512, 2.0, False, False, False),
}

# role -> candidate model aliases; order matters for the stable-hash pick (config.py:71-83)
DEFAULT_ROLE_MODELS = {
    "prompt_prep": ("qwen-7b", "llama-8b"),
    "retrieval": ("qwen-7b", "deepseek-7b"),
    "routing": ("qwen-7b",),
    "decomposition": ("deepseek-7b", "llama-8b"),
    "worker": ("qwen-7b", "deepseek-7b", "llama-8b"),
    "merge": ("llama-8b", "deepseek-7b"),
    "aggregation": ("llama-8b", "deepseek-7b"),
    "summarization": ("qwen-7b", "llama-8b"),
    "validation": ("deepseek-7b",),
    "verification": ("deepseek-7b", "qwen-7b"),
    "final_synthesis": ("llama-8b",),
}


def default_model_catalog() -> dict:
    return {
        alias: ModelProfile(alias, memory_gb=mem, prefill_coeff=pc, decode_coeff=dc,
                            switch_penalty=sw)
        for alias, mem, pc, dc, sw in _MODEL_ROWS
    }


def default_role_catalog() -> dict:
    out = {}
    for kind, (cx, pre, dec, mtok, otok, comm, keep, reuse, shard) in _ROLE_ROWS.items():
        out[kind] = StageRole(
            kind=kind, complexity=cx, prefill_scale=pre, decode_scale=dec,
            max_token_proxy=mtok, output_size_proxy=otok, comm_weight=comm,
            default_keep_cache=keep, default_cache_reuse=reuse, shard_eligible=shard,
        )
    return out


def default_topology(num_devices: int = 4) -> DeviceTopology:
    """``d0..d{n-1}``, unit speed, beta = 2.0 (reference config.py:86-88)."""
    return DeviceTopology(
        devices=tuple(DeviceSpec(id=f"d{i}", speed_factor=1.0) for i in range(num_devices)),
        default_transfer_coeff=2.0,
    )


_ABLATION_NAMES = ("no_future_planning", "no_locality", "no_same_model", "no_prefix", "no_shard")


@dataclass(frozen=True)
class AblationFlags:
    no_future_planning: bool = False
    no_locality: bool = False
    no_same_model: bool = False
    no_prefix: bool = False
    no_shard: bool = False

    def label(self) -> str:
        on = [name for name in _ABLATION_NAMES if getattr(self, name)]
        return "+".join(on) if on else "none"

    @staticmethod
    def from_names(names) -> "AblationFlags":
        unknown = sorted(set(names) - set(_ABLATION_NAMES))
        if unknown:
            raise ValueError(f"unknown ablation flags: {unknown}")
        return AblationFlags(**{name: True for name in names})


@dataclass(frozen=True)
class ScoreWeights:
    """Reference config.py:116-158; same defaults and validation."""

    lambda_q: float = 1.0
    lambda_s: float = 1.0
    lambda_tr: float = 1.0
    lambda_c: float = 0.5
    lambda_p: float = 0.5
    lambda_r: float = 0.5
    gamma: float = 0.5
    horizon: int = 4
    kappa_prefix: float = 1.0
    locality_coeff: float = 0.1
    shard_overhead_frac: float = 0.15
    demand_coeff: float = 0.6
    state_scale: float = 1.0
    locality_scale: float = 1.0
    prefix_scale: float = 1.0
    switch_x: float = 1.0
    transfer_x: float = 1.0
    prefix_x: float = 1.0
    ablation: AblationFlags = field(default_factory=AblationFlags)

    def __post_init__(self) -> None:
        for name in ("lambda_q", "lambda_s", "lambda_tr", "lambda_c", "lambda_p", "lambda_r"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        if not 0.0 < self.gamma <= 1.0:
            raise ValueError("gamma must be in (0, 1]")
        if self.horizon < 0:
            raise ValueError("horizon must be >= 0")
        for name in ("state_scale", "locality_scale", "prefix_scale",
                     "switch_x", "transfer_x", "prefix_x"):
            if not getattr(self, name) > 0:
                raise ValueError(f"{name} must be > 0")

    def effective_horizon(self) -> int:
        # no_future_planning keeps the solver but drops the tail (config.py:153-158)
        return min(self.horizon, 1) if self.ablation.no_future_planning else self.horizon


@dataclass(frozen=True)
class RunConfig:
    topology: DeviceTopology
    models: dict
    roles: dict
    role_models: dict
    weights: ScoreWeights

    def with_weights(self, weights: ScoreWeights) -> "RunConfig":
        return replace(self, weights=weights)


def default_config(num_devices: int = 4) -> RunConfig:
    return RunConfig(
        topology=default_topology(num_devices),
        models=default_model_catalog(),
        roles=default_role_catalog(),
        role_models=dict(DEFAULT_ROLE_MODELS),
        weights=ScoreWeights(),
    )
