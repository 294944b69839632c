"""Tooling parity on the GPU path: run_bench / BenchReport (bench.py:24-152) and PNM files."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2005_08713_b200")
from paper_2005_08713_b200 import synth  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_run_bench_corpus(tmp_path, oracle_lib):
    imgs = {"a_gray12.pgm": (synth.cfg1_gray12(3, 96).astype(np.int64), 12),
            "b_rgb.ppm": (synth.planar(synth.cfg2_pathology(4, 130, 200)).astype(np.int64), 8),
            "c_gray16.pgm": (np.random.default_rng(5).integers(0, 65536, (1, 33, 47)), 16)}
    for name, (a, bd) in imgs.items():
        P.write_pnm_file(P.RasterImage.from_planes(list(a), bd), tmp_path / name)
    (tmp_path / "b_rgb.png").write_bytes(b"\0" * 40000)
    (tmp_path / "notes.txt").write_text("ignored")
    rep = P.run_bench(tmp_path)
    assert [r.name for r in rep.rows] == sorted(imgs)
    for r in rep.rows:
        a, bd = imgs[r.name]
        ref = oracle_lib.encode_image(a, bd, P.default_levels(a.shape[2], a.shape[1]), a.shape[0] == 3)
        assert r.encoded_bytes == len(ref)
        assert r.pixels == a.shape[1] * a.shape[2] and r.encode_mps > 0 and r.decode_mps > 0
    assert rep.rows[1].ratio_vs_png == rep.rows[1].encoded_bytes / 40000
    assert len(rep.warnings) == 2 and rep.aggregate["images"] == 3
    assert "TOTAL" in rep.to_text() and rep.as_dict()["aggregate"]["ratio_vs_png"] > 0
    with pytest.raises(P.DomainError):
        P.run_bench(_empty(tmp_path))


def _empty(tmp_path):
    d = tmp_path / "empty"
    d.mkdir()
    return d


def test_pnm_roundtrip_through_codec(tmp_path):
    a = synth.planar(synth.cfg2_pathology(8, 77, 91)).astype(np.int64)
    P.write_pnm_file(P.RasterImage.from_planes(list(a), 8), tmp_path / "x.ppm")
    img = P.read_pnm_file(tmp_path / "x.ppm")
    data = P.encode_image(img, levels=3, use_rct=True)
    back = P.decode_image(data, level=1, planes_dropped=2)
    out = P.write_pnm(back, clamp=True)
    assert P.read_pnm(out).width == 46
