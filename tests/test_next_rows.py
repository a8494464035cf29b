"""Rows next to the path: Fredholm/GMRES solver, kernel SVM, CLI (reference: krylov.py, svm.py, cli.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REPO


def extras():
    with np.load(os.path.join(GOLDEN, "extras.npz")) as z:
        return {k: z[k] for k in z.files}


def test_synth_dataset_matches_reference_generator():
    from paper_2203_14832_b200.svm import synth_dataset

    g = extras()
    for shape, m, seed in (("rings2d", 300, 0), ("hypersphere4d", 257, 5)):
        ds = synth_dataset(shape, m, seed=seed)
        assert np.array_equal(ds.features, g[f"{shape}_features"])
        assert np.array_equal(ds.labels, g[f"{shape}_labels"])
        assert np.array_equal(ds.train_mask, g[f"{shape}_train"])


def test_cli_dry_run_and_usage():
    out = subprocess.run([sys.executable, "-m", "paper_2203_14832_b200", "matvec-bench", "--n-list", "1000",
                          "--dry-run"], cwd=REPO, capture_output=True, text=True)
    assert out.returncode == 0 and "n_list=[1000]" in out.stdout
    bad = subprocess.run([sys.executable, "-m", "paper_2203_14832_b200", "matvec-bench", "--n-list", "x"],
                         cwd=REPO, capture_output=True, text=True)
    assert bad.returncode == 2


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_14832_b200 as h2c

    return h2c


@pytest.mark.gpu
def test_fredholm_matches_reference(gpu):
    g = extras()
    rep, err, system = gpu.solve_fredholm(8, epsilon_nca=1e-7, epsilon_gmres=1e-10, seed=0)
    assert rep.converged
    assert abs(rep.iterations - int(g["fredholm8_iter"])) <= 1
    assert err <= 1e-6
    ref = g["fredholm8_solution"]
    assert np.linalg.norm(rep.solution - ref) / np.linalg.norm(ref) <= 1e-8
    hist = np.array(rep.residual_history)
    assert np.all(np.diff(hist) <= 1e-12)  # full GMRES: non-increasing


@pytest.mark.gpu
def test_gmres_identity_and_zero(gpu):
    b = np.random.default_rng(0).standard_normal(50)
    rep = gpu.gmres(lambda v: v, b, 1e-12)
    assert rep.iterations == 1 and np.allclose(rep.solution, b)
    rep0 = gpu.gmres(lambda v: v, np.zeros(10), 1e-12)
    assert rep0.iterations == 0 and rep0.converged


@pytest.mark.gpu
def test_gmres_dense_system(gpu):
    import torch

    rng = np.random.default_rng(1)
    A = np.eye(10) * 4 + rng.standard_normal((10, 10)) * 0.3
    b = rng.standard_normal(10)
    At = torch.as_tensor(A).cuda()
    rep = gpu.gmres(lambda v: At @ v, b, 1e-12)
    x = np.linalg.solve(A, b)
    assert np.linalg.norm(rep.solution - x) / np.linalg.norm(x) <= 1e-8


@pytest.mark.gpu
def test_svm_fast_and_dense_agree(gpu):
    from paper_2203_14832_b200.svm import synth_dataset, train

    data = synth_dataset("rings2d", 590, seed=3)
    k = gpu.builtin_kernel("matern", 2)
    mf, rf = train(data, k, backend="fast", max_iter=60, eps_nca=1e-8)
    md, rd = train(data, k, backend="dense", max_iter=60, eps_nca=1e-8)
    assert rf.iterations == rd.iterations
    assert np.linalg.norm(mf.alpha - md.alpha) / max(np.linalg.norm(md.alpha), 1e-300) <= 1e-5
    assert np.all(mf.alpha >= 0) and np.all(mf.alpha <= mf.lambda_box)


@pytest.mark.gpu
def test_svm_accuracy_and_model_roundtrip(gpu, tmp_path):
    from paper_2203_14832_b200.svm import evaluate, load_model, predict_batch, save_model, synth_dataset, train

    data = synth_dataset("rings2d", 3000, seed=0)
    model, rep = train(data, gpu.builtin_kernel("matern", 2), backend="fast", learn_rate=1e-4, max_iter=300)
    acc = evaluate(model, data)
    # the reference (h2cross, CPU) on the same call: OA 100.0, bias -0.7424828184605693, grad 0.35854331464718797
    assert acc["OA"] >= 99.0, acc
    assert model.bias == pytest.approx(-0.7424828184605693, rel=1e-6)
    assert rep.grad_norm == pytest.approx(0.35854331464718797, rel=1e-6)
    p = tmp_path / "m.txt"
    save_model(model, p)
    m2 = load_model(p)
    X, _ = data.test_split()
    assert np.array_equal(predict_batch(model, X[:50])[0], predict_batch(m2, X[:50])[0])


@pytest.mark.gpu
def test_cli_matvec_bench_runs(gpu, tmp_path):
    out = tmp_path / "mv.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2203_14832_b200", "matvec-bench", "--n-list", "2000,4000",
                        "--dim", "2", "--kernel", "matern", "--eps-nca", "1e-8", "-o", str(out)], cwd=REPO,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "N,mem,T_a,T_m,ε_m,max_rank" and len(lines) == 3
    assert all(float(ln.split(",")[4]) <= 1e-4 for ln in lines[1:]), lines
