"""Device accuracy evaluation vs the reference's own angular_error_map /
summarize (evaluation.py:34-73) on golden cases (tests/golden/make_golden_eval.py)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = __import__("pathlib").Path(__file__).resolve().parent / "golden" / "eval_cases.npz"
CASES = ["fixed9_all", "fixed9_ring", "adaptive_cd_all", "adaptive_cd_ring"]


@pytest.fixture(scope="module")
def ev():
    return np.load(GOLDEN)


@pytest.mark.parametrize("name", CASES)
def test_angular_error_and_stats(ev, cuda_dev, name):
    from paper_2504_15121_b200 import device
    est = np.where(ev[f"{name}__est_m"][..., None], ev[f"{name}__est_n"], np.nan)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda_dev)  # noqa: E731
    err, stats = device.angular_error(t(est), t(ev["gt_n"]), t(ev["gt_m"]),
                                      mask=t(ev[f"{name}__mask"]))
    e = err[0].cpu().numpy()
    ref = ev[f"{name}__err"]
    assert np.array_equal(np.isfinite(e), np.isfinite(ref))
    fin = np.isfinite(ref)
    assert np.abs(e[fin] - ref[fin]).max() < 1e-9
    s = stats[0].cpu().numpy()
    rs = ev[f"{name}__stats"]
    assert s[5] == rs[5]
    np.testing.assert_allclose(s[:5], rs[:5], rtol=1e-10, atol=1e-10)
    # summarize alone on the reference's own map: exact median / min / max
    s2 = device.error_stats(t(ref)[None])[0].cpu().numpy()
    assert s2[1] == rs[1] and s2[2] == rs[2] and s2[3] == rs[3] and s2[5] == rs[5]
    np.testing.assert_allclose(s2[[0, 4]], rs[[0, 4]], rtol=1e-12)


def test_reference_api_eval(ev, cuda_dev):
    import paper_2504_15121_b200 as sn
    name = "fixed9_ring"
    est = sn.NormalField(ev[f"{name}__est_n"], ev[f"{name}__est_m"])
    gt = sn.NormalField(ev["gt_n"], ev["gt_m"])
    err = sn.angular_error_map(est, gt, ev[f"{name}__mask"])
    st = sn.summarize(err)
    rs = ev[f"{name}__stats"]
    assert st.valid_count == int(rs[5])
    assert abs(st.median - rs[3]) < 1e-9 and abs(st.avg - rs[0]) < 1e-9
    st2 = sn.error_stats(est, gt, ev[f"{name}__mask"])
    assert st2.valid_count == int(rs[5]) and abs(st2.std - rs[4]) < 1e-9
    with pytest.raises(ValueError):
        sn.summarize(sn.ScalarField(np.full((4, 4), np.nan), np.zeros((4, 4), bool)))


@pytest.mark.parametrize("n", [1, 2, 3, 1000, 100001])
def test_error_stats_random(cuda_dev, n):
    """Lower median / population std on random maps incl. negatives, +-inf
    (invalid) and odd / even counts, batched."""
    from paper_2504_15121_b200 import device
    rng = np.random.default_rng(n)
    v = rng.normal(0, 10, (3, 1, n))
    v[0, 0, ::7] = np.nan
    v[1, 0, ::5] = np.inf
    out = device.error_stats(torch.from_numpy(v).to(cuda_dev)).cpu().numpy()
    for b in range(3):
        vals = v[b][np.isfinite(v[b])]
        if vals.size == 0:
            assert out[b, 5] == 0
            continue
        srt = np.sort(vals)
        assert out[b, 3] == srt[(len(srt) - 1) // 2]
        assert out[b, 1] == srt[0] and out[b, 2] == srt[-1] and out[b, 5] == vals.size
        np.testing.assert_allclose([out[b, 0], out[b, 4]], [vals.mean(), vals.std()], rtol=1e-12)


@pytest.mark.parametrize("kind", ["repeated", "all_equal", "narrow", "neg_zero"])
def test_error_stats_crowded(cuda_dev, kind):
    """Median prefixes holding more values than the candidate list (the
    8-bit radix fallback) and ones just below it, batched with a normal frame."""
    from paper_2504_15121_b200 import device
    rng = np.random.default_rng(7)
    n = 300007
    v = rng.normal(5, 2, (2, 1, n))
    if kind == "repeated":
        v[0, 0, : 2 * n // 3] = 1.25
    elif kind == "all_equal":
        v[0, 0, :] = 3.0
    elif kind == "narrow":  # ~all values share the top 24 key bits, distinct below
        v[0, 0, :] = 1.0 + rng.random(n) * 2.0 ** -20
    else:
        v[0, 0, :] = rng.choice([-0.0, 0.0, 1e-300, -1e-300], n)
    v[0, 0, ::11] = np.nan
    out = device.error_stats(torch.from_numpy(v).to(cuda_dev)).cpu().numpy()
    for b in range(2):
        vals = v[b][np.isfinite(v[b])]
        srt = np.sort(vals)
        med = srt[(len(srt) - 1) // 2]
        assert out[b, 3] == med or (med == 0 and out[b, 3] == 0), (kind, b, out[b, 3], med)
        assert out[b, 1] == srt[0] and out[b, 2] == srt[-1] and out[b, 5] == vals.size
        np.testing.assert_allclose([out[b, 0], out[b, 4]], [vals.mean(), vals.std()],
                                   rtol=1e-12, atol=1e-300)
