"""BASELINE config 4 (M = 4096, one instance) and the large path at M = 256,
against fixtures (tests/golden/large.npz, tests/golden/make_large.py):

  c4_heavy, c4_light   OG plan + IP-SSA solve at M = 4096 from the C oracle's
                       O(M^3 N) form (the reference's own og would need ~52
                       core-days here);
  ref256_heavy/light   OG plan + IP-SSA solve at M = 256 from the UNMODIFIED
                       reference (oracle/_ref), which also pins that oracle
                       form to the reference at this size.

CPU tests pin the oracle to the fixtures; GPU tests require the CUDA large
path (solve_large.cu) to reproduce every decision and energy bit."""
import numpy as np
import pytest

import checkers as ck
import golden_io

LARGE = golden_io.load_large()


@pytest.mark.parametrize("name", ["ref256_heavy", "ref256_light"])
def test_oracle_equals_reference_at_256(name):
    """The oracle's fast OG form equals the reference's og at M = 256."""
    c = LARGE[name]
    ck.assert_same_og(ck.oracle_og(c["profile"], c["users"], fast=True), c["og"], where=name)
    ck.assert_same_ip(ck.oracle_ipssa(c["profile"], c["users"]), c["ip"], where=name)


def test_oracle_reproduces_c4_heavy():
    """Regression pin of the C4 oracle (7 s): the fixture is its own output."""
    c = LARGE["c4_heavy"]
    ck.assert_same_og(ck.oracle_og(c["profile"], c["users"], fast=True), c["og"], where="c4_heavy")


def test_fixture_shapes():
    assert LARGE["c4_heavy"]["users"]["deadline"].shape == (1, 4096)
    assert LARGE["c4_light"]["og"]["n_groups"][0] == 80  # a long parent chain
    for c in LARGE.values():
        assert c["og"]["status"][0] == 0 and c["ip"]["status"][0] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(LARGE))
def test_large_path_bit_exact(engine, name):
    """OG plan (groups, bounds, splits, frequencies, per-user / per-group /
    total energies) and IP-SSA solve of the CUDA large path, bit for bit."""
    c = LARGE[name]
    ck.assert_same_og(engine.og(c["profile"], c["users"]), c["og"], where=name)
    ck.assert_same_ip(engine.ipssa(c["profile"], c["users"]), c["ip"], where=name)
    ip, og = engine.sweep(c["profile"], c["users"])  # fused path too
    ck.assert_same_og(og, c["og"], where=name + " sweep")
    ck.assert_same_ip(ip, c["ip"], where=name + " sweep")


@pytest.mark.gpu
def test_large_path_device_memory(engine):
    import torch
    c = LARGE["ref256_light"]
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in c["users"].items()}
    og = engine.og(c["profile"], dev)
    engine.synchronize()
    ck.assert_same_og({k: v.cpu().numpy() for k, v in og.items()}, c["og"], where="device")
