"""Config + sizing: mirror of kvsim.model for the hot path, plus the LLaMA-2
shapes the GPU runner executes.

Reference: /root/reference/pkg/src/kvsim/model.py.  Same dataclass names,
fields, defaults and validation errors (ConfigError(ValueError)):
  ModelProfile  model.py:92-127     TierConfig  model.py:130-153
  kv_size       model.py:243-247    prefill_time model.py:259-263
  preload_buffer_size model.py:273-287 (S_buf)
  parse_size / parse_bandwidth model.py:45-76, profile_from_dict / tiers_from_dict :323-359
Decimal units throughout (1 GB = 1e9 B), as in the reference.

B200-side additions: ``LlamaShape`` (layers, heads, head_dim, ffn) from which
the exact bf16 KV bytes/token follow (2 * L * Hkv * hd * 2), and
``profile_for(shape)`` building a ModelProfile whose kv_bytes_per_token is
that exact figure (the reference's built-in 13B profile uses a MiB-rounded
0.78e6, model.py:170).
"""

from __future__ import annotations

import re
from dataclasses import dataclass, fields, replace


class ConfigError(ValueError):
    """Invalid profile / tier configuration (model.py:21-22)."""


_UNITS = {"": 1, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12,
          "KIB": 2 ** 10, "MIB": 2 ** 20, "GIB": 2 ** 30, "TIB": 2 ** 40}
_NUM = re.compile(r"^\s*([0-9]*\.?[0-9]+(?:[eE][-+]?[0-9]+)?)\s*([A-Za-z]*)\s*$")


def parse_size(value) -> int:
    """'128GB', '0.78MB', '64MiB' or a number -> bytes (model.py:45-57)."""
    if isinstance(value, (int, float)):
        return int(value)
    m = _NUM.match(value)
    if not m:
        raise ConfigError(f"cannot parse size {value!r}")
    num, unit = m.groups()
    if unit.upper() not in _UNITS:
        raise ConfigError(f"unknown size suffix {unit!r} in {value!r}")
    return int(float(num) * _UNITS[unit.upper()])


def parse_bandwidth(value) -> float:
    """'26GB/s', '3.2GBps' or a number -> bytes/s (model.py:60-76)."""
    if isinstance(value, (int, float)):
        return float(value)
    text = value.strip()
    if text.lower().endswith("/s"):
        text = text[:-2]
    m = _NUM.match(text)
    if not m:
        raise ConfigError(f"cannot parse bandwidth {value!r}")
    num, unit = m.groups()
    unit = unit.upper().rstrip("P")
    if unit not in _UNITS:
        raise ConfigError(f"unknown bandwidth suffix in {value!r}")
    return float(num) * _UNITS[unit]


@dataclass(frozen=True)
class ModelProfile:
    name: str
    kv_bytes_per_token: float
    prefill_seconds_per_token: float
    decode_seconds_per_step: float
    context_window: int
    layers: int
    truncation_ratio: float = 0.5
    gpus: int = 1

    def __post_init__(self):
        checks = [
            (self.kv_bytes_per_token > 0, "kv_bytes_per_token must be positive"),
            (self.prefill_seconds_per_token > 0, "prefill_seconds_per_token must be positive"),
            (self.decode_seconds_per_step > 0, "decode_seconds_per_step must be positive"),
            (self.context_window >= 1, "context_window must be >= 1"),
            (self.layers >= 1, "layers must be >= 1"),
            (0.0 < self.truncation_ratio < 1.0, "truncation_ratio must lie in (0, 1)"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)

    @property
    def cut_tokens(self) -> int:
        """Truncation chunk max(1, int(ratio * W)) (sim.py:471, 578)."""
        return max(1, int(self.truncation_ratio * self.context_window))


@dataclass(frozen=True)
class TierConfig:
    hbm_exec_buffer: int = 40_000_000_000
    hbm_read_buffer: int = 10_000_000_000
    hbm_write_buffer: int = 10_000_000_000
    dram_capacity: int = 128_000_000_000
    disk_capacity: int = 10_000_000_000_000
    pcie_bandwidth: float = 26e9
    disk_bandwidth: float = 3.2e9

    def __post_init__(self):
        for n in ("hbm_exec_buffer", "hbm_read_buffer", "hbm_write_buffer", "dram_capacity",
                  "disk_capacity"):
            if getattr(self, n) < 0:
                raise ConfigError(f"{n} must be >= 0")
        if self.pcie_bandwidth <= 0 or self.disk_bandwidth <= 0:
            raise ConfigError("bandwidths must be positive")


def kv_size(tokens: int, profile: ModelProfile) -> float:
    if tokens < 0:
        raise ValueError("tokens must be >= 0")
    return tokens * profile.kv_bytes_per_token


def prefill_time(tokens: int, profile: ModelProfile) -> float:
    if tokens < 0:
        raise ValueError("tokens must be >= 0")
    return tokens * profile.prefill_seconds_per_token


def preload_buffer_size(hist_tokens: int, new_tokens: int, profile: ModelProfile,
                        tiers: TierConfig) -> float:
    """S_buf = B (T_load L_hist - T_pref L_new), floored at 0 (model.py:273-287)."""
    if hist_tokens < 0 or new_tokens < 0:
        raise ValueError("token counts must be >= 0")
    b = tiers.pcie_bandwidth
    gap = hist_tokens * profile.kv_bytes_per_token / b - new_tokens * profile.prefill_seconds_per_token
    return max(0.0, b * gap)


def profile_from_dict(raw: dict, base: ModelProfile | None = None) -> ModelProfile:
    """Build a profile from a mapping with human-readable sizes (model.py:323-345)."""
    raw = dict(raw)
    raw.pop("base", None)
    over = {k: (float(parse_size(v)) if k == "kv_bytes_per_token" else v) for k, v in raw.items()}
    if base is not None:
        return replace(base, **over)
    unknown = set(over) - {f.name for f in fields(ModelProfile)}
    if unknown:
        raise ConfigError(f"unknown profile fields: {sorted(unknown)}")
    try:
        return ModelProfile(**over)
    except TypeError as exc:
        raise ConfigError(f"incomplete profile definition: {exc}") from None


def tiers_from_dict(raw: dict) -> TierConfig:
    """model.py:348-359."""
    sizes = {"hbm_exec_buffer", "hbm_read_buffer", "hbm_write_buffer", "dram_capacity",
             "disk_capacity"}
    bws = {"pcie_bandwidth", "disk_bandwidth"}
    over = {}
    for k, v in raw.items():
        if k in sizes:
            over[k] = parse_size(v)
        elif k in bws:
            over[k] = parse_bandwidth(v)
        else:
            raise ConfigError(f"unknown tier field {k!r}")
    return TierConfig(**over)


# ---------------------------------------------------------------------------
# LLaMA-2 public shapes
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LlamaShape:
    name: str
    layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    context_window: int = 4096

    @property
    def row_elems(self) -> int:
        """bf16 elements of one token's K|V row in one layer: 2 * Hkv * hd."""
        return 2 * self.n_kv_heads * self.head_dim

    @property
    def row_bytes(self) -> int:
        return 2 * self.row_elems

    @property
    def kv_bytes_per_token(self) -> int:
        return self.layers * self.row_bytes

    @property
    def qkv_cols(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def params(self) -> int:
        attn = self.d_model * self.qkv_cols + self.n_heads * self.head_dim * self.d_model
        mlp = 3 * self.d_model * self.ffn
        return self.layers * (attn + mlp + 2 * self.d_model) + 2 * self.vocab * self.d_model

    def tp_shard(self, tp: int) -> "LlamaShape":
        """Per-rank shape under head-parallel TP."""
        if self.n_kv_heads % tp or self.n_heads % tp or self.ffn % tp:
            raise ConfigError(f"{self.name} does not shard over tp={tp}")
        return replace(self, name=f"{self.name}/tp{tp}", n_heads=self.n_heads // tp,
                       n_kv_heads=self.n_kv_heads // tp, ffn=self.ffn // tp)


SHAPES = {
    "tiny": LlamaShape("tiny", 2, 256, 4, 4, 64, 512, 512),
    "llama2-7b": LlamaShape("llama2-7b", 32, 4096, 32, 32, 128, 11008, 32000),
    "llama2-13b": LlamaShape("llama2-13b", 40, 5120, 40, 40, 128, 13824, 32000),
    "llama2-70b": LlamaShape("llama2-70b", 80, 8192, 64, 8, 128, 28672, 32000),
}
ALIASES = {"7b": "llama2-7b", "13b": "llama2-13b", "70b": "llama2-70b"}


def shape(name: str) -> LlamaShape:
    try:
        return SHAPES[ALIASES.get(name, name)]
    except KeyError:
        raise ConfigError(f"unknown shape {name!r} (known: {sorted(SHAPES)})") from None


def profile_for(s: LlamaShape, *, prefill_seconds_per_token: float = 1e-4,
                decode_seconds_per_step: float = 1e-3, truncation_ratio: float = 0.5,
                gpus: int = 1) -> ModelProfile:
    return ModelProfile(name=s.name, kv_bytes_per_token=float(s.kv_bytes_per_token),
                        prefill_seconds_per_token=prefill_seconds_per_token,
                        decode_seconds_per_step=decode_seconds_per_step,
                        context_window=s.context_window, layers=s.layers,
                        truncation_ratio=truncation_ratio, gpus=gpus)
