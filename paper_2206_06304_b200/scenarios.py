"""Synthetic problem inputs (the input side of the hot path).

Profiles are built exactly like the reference (synth_profile / profile_heavy /
profile_light, scenario_gen.hpp:182-216): F_n(b) = base_n*(1+growth_n*(b-1))
with the same two rounded operations, so the tables are bit-identical.

`sample_batch` draws scenarios with the distribution of sample_scenario
(scenario_gen.hpp:113-173, ScenarioConfig defaults :49-63): users uniform on a
100 m disk (>= 1 m from the antenna), 3GPP path loss 128.1+37.6 log10(d_km)
plus N(0, 8 dB) shadowing, Shannon rate over 1 MHz, devices calibrated by
calibrate_device (core_model.hpp:147-151), deadlines uniform and redrawn below
the all-local floor.  It uses numpy's generator, not libstdc++'s, so the bits
differ from the reference generator's; parity never depends on that because
the CUDA engine and the checkers always consume the same input bytes.
"""
from __future__ import annotations

import math
from typing import Dict

import numpy as np

from .engine import ProfileArrays

HEAVY = dict(base=[0.030, 0.020, 0.015, 0.010], growth=[0.12] * 4,
             bits=[2e6, 4e5, 3e5, 2e5, 1e5])
LIGHT = dict(base=[0.004, 0.003, 0.002, 0.001], growth=[0.0] * 4,
             bits=[1.5e5, 8e4, 5e4, 3e4, 1e4])


def synth_profile(base, growth, bits, b_max: int) -> ProfileArrays:
    base = np.asarray(base, dtype=np.float64)
    growth = np.asarray(growth, dtype=np.float64)
    b = np.arange(b_max, dtype=np.float64)  # b - 1
    lat = base[:, None] * (1.0 + growth[:, None] * b[None, :])
    return ProfileArrays(base.copy(), np.asarray(bits, dtype=np.float64), np.ascontiguousarray(lat))


def profile_heavy(b_max: int = 15) -> ProfileArrays:
    return synth_profile(HEAVY["base"], HEAVY["growth"], HEAVY["bits"], b_max)


def profile_light(b_max: int = 15) -> ProfileArrays:
    return synth_profile(LIGHT["base"], LIGHT["growth"], LIGHT["bits"], b_max)


def sample_batch(n_inst: int, M: int, profile: ProfileArrays, low: float = 0.25,
                 high: float = 1.0, seed: int = 1, bandwidth: float = 1e6,
                 cell_radius: float = 100.0, shadow_sigma_db: float = 8.0,
                 tx_power: float = 0.05, noise_dbm_hz: float = -174.0, uplink_power: float = 1.0,
                 edge_power: float = 300.0, rho: float = 1.0, alpha: float = 1.0) -> Dict[str, np.ndarray]:
    rng = np.random.default_rng(seed)
    shape = (n_inst, M)
    r = cell_radius * np.sqrt(rng.random(shape))
    bad = r < 1.0
    while bad.any():  # area-uniform radius, >= 1 m off the antenna
        r[bad] = cell_radius * np.sqrt(rng.random(int(bad.sum())))
        bad = r < 1.0
    sh = rng.normal(0.0, shadow_sigma_db, shape) if shadow_sigma_db > 0 else np.zeros(shape)
    pl = 128.1 + 37.6 * np.log10(r / 1000.0) + sh
    gain = np.power(10.0, -pl / 10.0)
    noise = math.pow(10.0, (noise_dbm_hz - 30.0) / 10.0)
    snr = tx_power * gain / (bandwidth * noise)
    rate = bandwidth * np.log2(1.0 + snr)
    f_max = 1.0 / alpha
    kappa = rho * edge_power * alpha * alpha
    floor = float(profile.work.sum()) / f_max
    if low == high:
        dl = np.full(shape, float(low))
    else:
        dl = rng.uniform(low, high, shape)
        bad = dl < floor
        while bad.any():
            dl[bad] = rng.uniform(low, high, int(bad.sum()))
            bad = dl < floor
    one = np.ones(shape)
    return dict(f_min=np.zeros(shape), f_max=one * f_max, kappa=one * kappa, rate_up=rate,
                power_up=one * uplink_power, arrival=np.zeros(shape), deadline=dl,
                rate_down=rate.copy(), power_down=one * uplink_power)


def _mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer (ddpg.hpp:272-277), vectorised over uint64."""
    x = (x + np.uint64(0x9e3779b97f4a7c15)).astype(np.uint64)
    x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)).astype(np.uint64)
    x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94d4a9749d57afbb)).astype(np.uint64)
    return x ^ (x >> np.uint64(31))


def sub_seed(root: int, component: int, index) -> np.ndarray:
    """The CLI's per-stream seeds (coinfer_main.cpp:47-50):
    mix64(mix64(root ^ component * golden) + index), vectorised over index."""
    with np.errstate(over="ignore"):
        r = np.uint64(root) ^ (np.uint64(component) * np.uint64(0x9e3779b97f4a7c15))
        base = _mix64(np.array([r], dtype=np.uint64))[0]
        idx = np.asarray(index, dtype=np.uint64)
        return _mix64((base + idx).astype(np.uint64))
