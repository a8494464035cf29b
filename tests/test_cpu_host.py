"""CPU-only checks: the C ABI library loads and exports every declared symbol,
host-side logic mirrors the reference, sampling matches the reference's."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO, load_golden


def header_symbols():
    text = open(os.path.join(REPO, "include", "h2b.h")).read()
    return sorted(set(re.findall(r"\b(h2b_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2203_14832_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.h2b_version() == 1


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2203_14832_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert not re.search(r"(from|import)\s+oracle|h2oracle|oh2_", text), f


def test_gpu_call_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    import paper_2203_14832_b200 as h2c

    cloud = h2c.PointCloud.from_points(np.random.default_rng(0).uniform(-1, 1, (100, 2)))
    with pytest.raises(Exception):
        h2c.build_tree(cloud, nu=16, eta=1.4)


def test_pointcloud_and_kernel_registry():
    import paper_2203_14832_b200 as h2c

    with pytest.raises(ValueError):
        h2c.PointCloud(np.zeros((3, 2)), np.zeros((3, 3)))
    with pytest.raises(ValueError, match="unknown kernel"):
        h2c.builtin_kernel("helmholtz", 3)
    k = h2c.builtin_kernel("gaussian", 3, sigma=0.5)
    assert k.kind == 7 and k.device_param == 2.0
    assert h2c.builtin_kernel("gaussian", 3).kind == 4
    assert h2c.builtin_kernel("laplace-3d", 3).evaluate(np.zeros(3), np.array([0.0, 0.0, 2.0])) == \
        pytest.approx(1 / (8 * np.pi))
    assert h2c.relative_error([3.0, 4.0], [0.0, 5.0]) == pytest.approx(np.sqrt(10) / 5)
    with pytest.raises(ValueError):
        h2c.relative_error([1.0], [0.0])


def test_python_admissibility_matches_reference_goldens():
    from paper_2203_14832_b200.geometry import boxes_admissible
    from conftest import GOLDEN

    with np.load(os.path.join(GOLDEN, "aca_blocks.npz")) as z:
        C, HW, R = z["adm_c"], z["adm_hw"], z["adm_res"]
    for row, hw, res in zip(C[:1500], HW, R):
        d = int(row[0])
        assert boxes_admissible(row[1:1 + d], hw, row[5:5 + d], hw, float(np.sqrt(2.0))) == bool(res)


def test_sampling_matches_reference_generators():
    from paper_2203_14832_b200 import sampling

    g = load_golden("u2d_reglog")
    assert np.array_equal(sampling.uniform_points(4096, 2, 0), g["P"])
    g = load_golden("cheb2d_reginv")
    assert np.array_equal(sampling.chebyshev_points(1024, 2, 0), g["P"])
    s = sampling.sphere_points(1000, 3, 2)
    assert np.allclose(np.linalg.norm(s, axis=1), 1.0)


def test_bench_reference_arm_contract():
    """bench.py --impl reference: the CPU reference path (oracle) prints one JSON line with the contract keys."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--impl", "reference", "--config", "c0",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "N^2/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["steps"] == 1 and line["warmup"] == 3
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["N"] == 4096
