"""DVFS domain and device constants — host mirror of the reference types.

DeviceConstants / DvfsDomain follow proj/include/dso/dvfs_model.hpp:36-42 and
proj/include/dso/optimizer.hpp:14-18; default_device / default_domain follow
proj/src/sim_harness.cpp:103-116; the benchmark domains are the ones
BASELINE.json's configs name.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class DeviceConstants:
    kappa_vf: float
    pmax_w: float
    vmin_v: float
    vmax_v: float
    mhz_per_unit: float

    def as_array(self) -> np.ndarray:
        return np.array([self.kappa_vf, self.pmax_w, self.vmin_v, self.vmax_v,
                         self.mhz_per_unit], dtype=np.float64)


@dataclass
class DvfsDomain:
    core_freqs_mhz: np.ndarray
    mem_freqs_mhz: np.ndarray
    dev: DeviceConstants = field(default_factory=lambda: default_device())

    def __post_init__(self):
        self.core_freqs_mhz = np.asarray(self.core_freqs_mhz, dtype=np.float64)
        self.mem_freqs_mhz = np.asarray(self.mem_freqs_mhz, dtype=np.float64)

    @property
    def nc(self) -> int:
        return len(self.core_freqs_mhz)

    @property
    def nm(self) -> int:
        return len(self.mem_freqs_mhz)

    @property
    def pairs(self) -> int:
        return self.nc * self.nm

    def vc(self) -> np.ndarray:
        """required_voltage_mhz per core level (dvfs_model.hpp:117-128)."""
        d = self.core_freqs_mhz / self.dev.mhz_per_unit - self.dev.kappa_vf
        return 2.0 * d * d + self.dev.kappa_vf

    def config_of(self, idx: int):
        """(vc, fc, fm) of grid index idx = fc_idx * nm + fm_idx."""
        i, j = divmod(int(idx), self.nm)
        return float(self.vc()[i]), float(self.core_freqs_mhz[i]), float(self.mem_freqs_mhz[j])


def validate_domain(domain: DvfsDomain) -> None:
    """validate(DvfsDomain) (optimizer.cpp:58-88), run by the library's host code."""
    import ctypes as C

    from ._lib import DsoError, lib, status_kind
    core = np.ascontiguousarray(domain.core_freqs_mhz, np.float64)
    mem = np.ascontiguousarray(domain.mem_freqs_mhz, np.float64)
    dev = domain.dev.as_array()
    dp = C.POINTER(C.c_double)
    buf = C.create_string_buffer(512)
    st = lib().dso_validate_domain(core.ctypes.data_as(dp), len(core), mem.ctypes.data_as(dp),
                                   len(mem), dev.ctypes.data_as(dp), buf, 512)
    if st:
        raise DsoError(status_kind(st), buf.value.decode())


def default_device() -> DeviceConstants:
    """sim_harness.cpp:103-106."""
    return DeviceConstants(kappa_vf=0.5, pmax_w=300.0, vmin_v=0.55, vmax_v=2.10,
                           mhz_per_unit=1000.0)


def default_domain() -> DvfsDomain:
    """sim_harness.cpp:108-116: 705 + 52k (k < 13) and 1380 MHz x {438, 658, 877}."""
    core = [705.0 + 52.0 * k for k in range(13)] + [1380.0]
    return DvfsDomain(np.array(core), np.array([438.0, 658.0, 877.0]), default_device())


def linear_domain(nc: int, nm: int) -> DvfsDomain:
    """Benchmark grids: fc = 705 + 675 i/(nc-1); fm = 438 + 439 j/(nm-1),
    or {877} when nm == 1."""
    core = 705.0 + (1380.0 - 705.0) * np.arange(nc) / max(nc - 1, 1)
    mem = np.array([877.0]) if nm == 1 else 438.0 + 439.0 * np.arange(nm) / (nm - 1)
    return DvfsDomain(core, mem, default_device())


def config_domain(name: str) -> DvfsDomain:
    """Domains of BASELINE.json's configs: c1 (default 14x3), c1_literal (10x1),
    c2 (64x1), c3 / c4 (128x4)."""
    name = name.lower()
    if name == "c1":
        return default_domain()
    if name == "c1_literal":
        return DvfsDomain(705.0 + 75.0 * np.arange(10), np.array([877.0]), default_device())
    if name == "c2":
        return linear_domain(64, 1)
    if name in ("c3", "c4"):
        return linear_domain(128, 4)
    raise ValueError(f"unknown config {name!r}")
