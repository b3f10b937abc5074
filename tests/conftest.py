import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")


def _load(name):
    z = np.load(GOLDEN / name, allow_pickle=False)
    names = [str(n) for n in z["names"]]
    cases = {}
    for n in names:
        pre = f"{n}__"
        cases[n] = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
    return cases


@pytest.fixture(scope="session")
def fixed_golden():
    return _load("fixed_cases.npz")


@pytest.fixture(scope="session")
def ccl_golden():
    return _load("ccl_cases.npz")


@pytest.fixture(scope="session")
def cuda_dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def adaptive_golden():
    import json
    z = np.load(GOLDEN / "adaptive_cases.npz", allow_pickle=False)
    out = {}
    for n, c in zip([str(v) for v in z["names"]], [str(v) for v in z["configs"]]):
        pre = f"{n}__"
        case = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
        case["config"] = json.loads(c)
        out[n] = case
    return out


@pytest.fixture(scope="session")
def codec_golden():
    z = np.load(GOLDEN / "codec_cases.npz", allow_pickle=False)
    out = {"pfm": {}, "png": {}, "fused": {}}
    for kind in out:
        for n in [str(v) for v in z[f"{kind}_names"]]:
            pre = f"{kind}_{n}__"
            out[kind][n] = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
    out["pfmerr"] = [(bytes(z[f"pfmerr_{i}__bytes"]), str(m))
                     for i, m in enumerate(z["pfmerr_msgs"])]
    return out


@pytest.fixture(scope="session")
def f64_golden():
    """tests/golden/f64_cases.npz (make_golden_f64.py): reference outputs on
    float64 inputs; frames are regenerated from their seeds (f64_input)."""
    import json
    z = np.load(GOLDEN / "f64_cases.npz", allow_pickle=False)
    arrays = {k: z[k] for k in z.files if k != "meta"}
    meta = json.loads(str(z["meta"]))
    return meta, arrays


_INPUTS = {}


def f64_input(entry):
    """The float64 street frame of a golden entry (SURVEY.md §8(d) recipe),
    regenerated and checked against the recorded SHA-256."""
    import hashlib
    key = (entry["w"], entry["h"], entry["sigma"], entry["seed"], entry["holes"])
    if key not in _INPUTS:
        from scipy import ndimage
        from paper_2504_15121_b200 import scenes
        sc = scenes.street_scene(entry["w"], entry["h"])
        d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], entry["sigma"], entry["seed"])
        if entry["holes"]:
            m = ndimage.binary_dilation(
                np.random.default_rng(1000 + entry["seed"]).random(d.shape) < 0.002, iterations=3)
            d = np.where(m, np.nan, d)
        got = hashlib.sha256(np.ascontiguousarray(d, dtype=np.float64).tobytes()).hexdigest()
        assert got == entry["sha256"], f"regenerated input differs from the golden's ({entry})"
        _INPUTS[key] = (d, sc.rig)
    return _INPUTS[key]
