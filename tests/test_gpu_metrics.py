"""Reconstruction metrics on the GPU (pdf_relative_error, pdf_count_components;
reference reconstruct.py:243-254) against the reference's own outputs
(tests/golden/make_golden.py `metrics`) and its unit tests
(tests/test_reconstruct.py:102-113, tests/test_scenes.py:71-74)."""
import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g_metrics():
    return golden("metrics")


def test_count_components_matches_reference(g_metrics):
    from paper_2602_13805_b200.metrics import count_components
    g = g_metrics
    thr = float(g["thr"])
    for k, want in enumerate(g["counts"]):
        assert count_components(g[f"img{k}"] + 1.0, thr) == want, (k, g[f"img{k}"].shape)
    for k, want in enumerate(g["extra_counts"]):       # serpentine, checkerboard, austria preset, empty, full
        assert count_components(g[f"extra{k}"] + 1.0, thr) == want, k


def test_count_components_batched_and_complex(g_metrics):
    """A stack of complex contrast images in one launch (offset 1: eps = chi + 1)."""
    from paper_2602_13805_b200.metrics import count_components_dev
    g = g_metrics
    ks = [k for k in range(len(g["counts"])) if g[f"img{k}"].shape == (64, 64)]
    chi = np.stack([g[f"img{k}"].astype(float) + 0.3j for k in ks])
    got = count_components_dev(torch.as_tensor(chi, device="cuda"), float(g["thr"]), offset=1.0).cpu().numpy()
    assert list(got) == [int(g["counts"][k]) for k in ks]


def test_reference_unit_cases():
    from paper_2602_13805_b200.metrics import count_components, relative_error
    img = np.zeros((6, 6))
    img[1, 1] = img[2, 2] = 2.0
    img[4, 4] = img[4, 5] = 2.0
    assert count_components(img, 1.5) == 3
    a, b = np.full((4, 4), 2.0), np.full((4, 4), 1.0)
    assert relative_error(a, b) == pytest.approx(1.0)
    assert relative_error(b, b) == 0.0


def test_relative_error_matches_reference(g_metrics):
    from paper_2602_13805_b200.metrics import relative_error, relative_error_dev
    g = g_metrics
    for k, want in enumerate(g["rels"]):
        assert abs(relative_error(g["rel_a"][k].real + 1.0, g["rel_b"][k].real + 1.0) - want) < 1e-14
    got = relative_error_dev(torch.as_tensor(g["rel_a"], device="cuda"), torch.as_tensor(g["rel_b"], device="cuda"),
                             offset=1.0).cpu().numpy()
    np.testing.assert_allclose(got, g["rels"], rtol=1e-14)
