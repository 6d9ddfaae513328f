"""Host logic of bench.py (no GPU): the kernel each config's bench line names (it mirrors the C-ABI
dispatch) and the algorithmic bytes behind roofline.achieved."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2301_12457_b200 import workloads as WL  # noqa: E402


@pytest.mark.parametrize("cfg,kernel", [("H", "k_pso_gen_wave<ackley>"), ("C1", "k_pso_run_small<sphere>"),
                                        ("C2", "k_pso_run_mid<ackley>"), ("C3", "k_cso_gen<rastrigin>"),
                                        ("C4g", "k_pso_gen_flat<griewank>"),
                                        ("C4r", "k_pso_gen_flat<rosenbrock>"), ("C5", "k_pso_gen_wave<ackley>"),
                                        ("D1", "k_de_gen_flat<sphere>"), ("D2", "k_de_gen<ackley>")])
def test_kernel_names(cfg, kernel):
    c = WL.CONFIGS[cfg]
    assert bench.gen_kernel_name(c, c.pop, 1) == kernel


def test_kernel_name_wave_threshold():
    """Warp-per-row rows take the wave grid only from 3 waves of 8-row CTAs."""
    few = WL.Config("x", "pso", "ackley", 10_000, 4096, 1, "")
    many = WL.Config("x", "pso", "ackley", 40_000, 4096, 1, "")
    assert bench.gen_kernel_name(few, few.pop, 1) == "k_pso_gen<ackley>"
    assert bench.gen_kernel_name(many, many.pop, 1) == "k_pso_gen_wave<ackley>"
    grie = WL.Config("x", "pso", "griewank", 1_000_000, 1000, 1, "")
    assert bench.gen_kernel_name(grie, grie.pop, 1) == "k_pso_gen<griewank>"


def test_algorithmic_bytes():
    """SURVEY §8(a)/(d) per-element and per-row bytes."""
    h = WL.CONFIGS["H"]
    assert bench.algorithmic_bytes(h, h.pop) == 20 * 1000 * 10**6 + 10 * 10**6
    c3 = WL.CONFIGS["C3"]
    assert bench.algorithmic_bytes(c3, c3.pop) == 10 * 1000 * 10**5 + 6 * 10**5
    d1 = WL.CONFIGS["D1"]
    assert bench.algorithmic_bytes(d1, d1.pop) == 20 * 100 * 10**6 + 13 * 10**6
    e = WL.CONFIGS["EH-ackley"]
    assert bench.algorithmic_bytes(e, e.pop) == 4 * 1000 * 10**6 + 4 * 10**6


def test_config_dict_same_in_both_arms():
    """The reference arm prints the GPU arm's config dict (the driver compares them)."""
    c = WL.CONFIGS["H"]
    d = bench.config_dict(c, 1, "peer")
    assert d["workload"] == c.note and d["pop"] == c.pop and d["dim"] == c.dim
    assert {"seed", "parallelism", "l2"} <= set(d)
