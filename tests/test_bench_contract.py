"""bench.py's work model and roofline bookkeeping (no GPU): the bound each
kernel is reported against and the units of its roofline object."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


PK = {"hbm_gbs": 6547.2, "sm_max_mhz": 1965.0, "bf16_tflops": 1668.7, "src": "test"}


def test_passes_are_mufu_bound_reported_as_alu(bench):
    N, m, d = 4194304, 256, 16
    for name in ("rfd_pass1_tc", "rfd_pass2_tc"):
        rl = bench.roofline_of(name, N, m, d, 0.75, PK)
        assert rl["bound"] == "alu" and rl["pipe"] == "mufu" and rl["unit"] == "Tops/s"
        # 2m sin/cos per point at 148 x 16 / clk
        t = 2.0 * N * m / (148 * 16 * 1965e6)
        assert abs(rl["frac"] - t / 0.75e-3) < 1e-9
        assert abs(rl["achieved"] / rl["peak"] - rl["frac"]) < 1e-9


def test_gram_over_grid_nodes_is_tensor_bound(bench):
    N, m, d, nodes = 4194304, 256, 16, 67445
    rl = bench.roofline_of("rfd_gram_tc", N, m, d, 0.07, PK, nodes)
    assert rl["bound"] == "tensor" and rl["unit"] == "TFLOP/s"
    r = 2 * m
    assert abs(rl["achieved"] - 2.0 * nodes * r * (r + 1) / 2 / 0.07e-3 / 1e12) < 1e-6
    # without the grid the same call counts the N points
    rl_direct = bench.roofline_of("rfd_gram_tc", N, m, d, 2.76, PK)
    assert rl_direct["bound"] == "tensor"
    assert rl_direct["achieved"] > rl["achieved"] * 0.5


def test_bound_vocabulary(bench):
    for name, nodes in (("rfd_pass1_tc", 0), ("rfd_pass2_tc", 0), ("rfd_gram_tc", 0),
                        ("rfd_gram_tc", 50000), ("rfd_nufft_spread", 50000)):
        rl = bench.roofline_of(name, 1 << 22, 256, 16, 0.5, PK, nodes)
        assert rl["bound"] in ("hbm", "tensor", "alu"), (name, rl["bound"])
        assert rl["unit"] in ("GB/s", "TFLOP/s", "Tops/s")
    assert bench.roofline_of("rfd_core_dgemm", 1 << 22, 256, 16, 0.02, PK) is None
