"""Runtime configuration (mirror of cl/config.py:79-176, B200 semantics).

Same keys as the reference's RuntimeConfig so callers and TOML files carry
over. Differences, all deliberate:
  * time_mode defaults to "wall": on real HBM/NVLink there is nothing to
    model, so the reference's virtual clock (cl/config.py:84,
    cl/timebase.py:14-31) is rejected with a ConfigError;
  * link/copy cost models are accepted for compatibility and ignored;
  * device_capacity defaults to None (= the GPU's free HBM);
  * ``gpus`` maps worker -> CUDA ordinal (default: worker % device_count).
"""

from __future__ import annotations

import sys
from dataclasses import dataclass, field, replace

if sys.version_info >= (3, 11):
    import tomllib as _toml
else:  # pragma: no cover
    import tomli as _toml

WALL = "wall"
VIRTUAL = "virtual"


class ConfigError(ValueError):
    pass


@dataclass(frozen=True)
class LinkModel:
    """Accepted for API compatibility (cl/config.py:25-50); unused on GPU."""

    latency_us: float = 1.0
    bandwidth_gbps: float = 12.5


@dataclass(frozen=True)
class CopyCostModel:
    """Accepted for API compatibility (cl/config.py:53-66); unused on GPU."""

    h2d_latency_us: float = 5.0
    h2d_bandwidth: float = 10e9
    d2h_latency_us: float = 5.0
    d2h_bandwidth: float = 10e9


@dataclass(frozen=True)
class TagLayoutSpec:
    """Field widths of the 64-bit tag (cl/config.py:69-76)."""

    pe_bits: int = 32
    counter_bits: int = 28
    channel_id_bits: int = 28
    channel_counter_bits: int = 32


@dataclass
class RuntimeConfig:
    """Top-level configuration (cl/config.py:79-107)."""

    workers: int = 1
    time_mode: str = WALL
    eager_threshold: int = 8192
    eager_prepost: int = 64
    max_message_bytes: int = 1 << 30
    connect_timeout_s: float = 5.0
    ranks_per_node: int = 1
    seed: int = 0
    addresses: dict = field(default_factory=dict)
    link_intra: LinkModel = field(default_factory=lambda: LinkModel(1.0, 50.0))
    link_inter: LinkModel = field(default_factory=LinkModel)
    copy_model: CopyCostModel = field(default_factory=CopyCostModel)
    device_capacity: int | None = None
    tag_layout: TagLayoutSpec = field(default_factory=TagLayoutSpec)
    gpus: tuple | None = None  # worker -> CUDA ordinal; None = round robin
    flag_timeout_s: float = 30.0  # device-side wait bound (never hang a GPU)
    # "loopback": every PE in this process; "ipc": one process per GPU under
    # torch.distributed, PE p in process p % world (transport.TransportGroup)
    backend: str = "loopback"

    def __post_init__(self):
        self.validate()

    def validate(self) -> None:
        if self.time_mode == VIRTUAL:
            raise ConfigError(
                "time_mode='virtual' models the reference's simulated device space; the B200 "
                "path moves real bytes and is timed with wall clocks / CUDA events")
        if self.time_mode != WALL:
            raise ConfigError(f"time_mode must be 'wall', got {self.time_mode!r}")
        if self.workers < 1:
            raise ConfigError("workers must be >= 1")
        if self.backend not in ("loopback", "ipc"):
            raise ConfigError(f"backend must be 'loopback' or 'ipc', got {self.backend!r}")

    def node_of(self, rank: int) -> int:
        return rank // max(1, self.ranks_per_node)

    def with_overrides(self, **kw) -> "RuntimeConfig":
        cfg = replace(self, **kw)
        cfg.validate()
        return cfg


def load_config(path: str) -> RuntimeConfig:
    """TOML loader with the reference's keys (cl/config.py:115-126)."""
    with open(path, "rb") as f:
        raw = _toml.load(f)
    return config_from_dict(raw)


def config_from_dict(raw: dict) -> RuntimeConfig:
    kw = {}
    for key, conv in (("workers", int), ("time_mode", str), ("eager_threshold", int),
                      ("eager_prepost", int), ("ranks_per_node", int), ("seed", int),
                      ("connect_timeout_s", float)):
        if key in raw:
            kw[key] = conv(raw[key])
    kw.setdefault("time_mode", WALL)
    if "addresses" in raw:
        kw["addresses"] = {int(k): str(v) for k, v in raw["addresses"].items()}
    dev = raw.get("device", {})
    if "capacity_gib" in dev:
        kw["device_capacity"] = int(float(dev["capacity_gib"]) * (1 << 30))
    if "gpus" in dev:
        kw["gpus"] = tuple(int(g) for g in dev["gpus"])
    tags = raw.get("tags", {})
    if tags:
        kw["tag_layout"] = TagLayoutSpec(**{k: int(v) for k, v in tags.items()})
    return RuntimeConfig(**kw)
