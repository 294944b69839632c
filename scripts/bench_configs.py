"""Device throughput of every BASELINE config on one GPU (developer tool; the driver's headline is
bench.py on configs[3], the whole slide).  Writes one JSON object to stdout.

cfg1  1 x 512^2 gray12, L3: batch of 64 images (latency-bound alone), encode / decode / round trip
cfg2  2048^2 RGB8, RCT, L4: batch of 8 (the bench.py workload, single stream here)
cfg3  4096^2 RGB8, RCT, L5, lossy: encode, device truncate n=2 / n=4, decode; PSNR vs the input
cfg4  4096^2 RGB8 tiles, RCT, L6: 8 tiles per GPU pass (a 65536^2 slide = 256 tiles: 32 per GPU
      at 8 GPUs, weak scaling); slide MP/s on one GPU = tiles/s x 16.78 MP
cfg5  4 x 8192^2 u16, L5: decode only (container from this encoder; bit-exact with the reference
      per tests/test_gpu_parity.py::test_cfg5_fluorescence)

Times are CUDA events on the launching stream, median of `--iters` after warm-up, L2 flushed
(256 MB write) before each timed call.  DWT level-1 kernel rooflines come from the library's
per-kernel event marks.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2005_08713_b200 as P  # noqa: E402
from paper_2005_08713_b200 import _lib, synth  # noqa: E402
from paper_2005_08713_b200.container import Codec, ContainerHeader  # noqa: E402

FLUSH = None


def timed(fn, iters):
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(iters):
        FLUSH.fill_(i & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def kernel_us(fn, iters):
    _lib.profile_enable(True)
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    _lib.profile_enable(False)
    return {k: round(ms / n * 1e3, 1) for k, (ms, n) in prof.items()}


def codec_case(name, x, W, H, C, bd, L, rct, layout, iters, peak):
    B = x.shape[0]
    codec = Codec(W, H, C, bd, L, rct, x.dtype, layout, batch=B)
    codec.roundtrip_device(x)
    codec.check()
    assert torch.equal(codec.pixels_out, x), f"{name}: round trip mismatch"
    mp = B * W * H / 1e6
    te = timed(lambda: codec.encode_device(x), iters)
    td = timed(lambda: codec.decode_device(), iters)
    tr = timed(lambda: codec.roundtrip_device(x), iters)
    ku = kernel_us(lambda: codec.roundtrip_device(x), iters)
    sizes = codec.container_sizes()
    elem = x.element_size()
    out = {"images": B, "mp_per_step": round(mp, 2), "encode_mps": round(mp / te * 1e3, 1),
           "decode_mps": round(mp / td * 1e3, 1), "roundtrip_mps": round(mp / tr * 1e3, 1),
           "encode_ms": round(te, 3), "decode_ms": round(td, 3),
           "compression_ratio": round(B * W * H * C * elem / sum(sizes), 3), "kernel_us": ku}
    # DWT rooflines: level 1 alone (samples in/out + the level-1 planes it moves) and all levels
    # together (compulsory C*(s_in + s_coef) per pixel forward, C*(s_coef + s_out)
    # inverse), coefficients at the stored width (encode: coef_bytes; decode details: int16 when
    # the encoder's int16 bound holds, the level-1 LL plane the last inverse level reads is int32)
    n = B * W * H * C
    s_det = 2 if codec.coef_bytes == 2 else 4
    cnt = {k: v for k, v in kernel_counts(lambda: codec.roundtrip_device(x)).items()}
    if "dwt_fwd_l1" in ku:
        a = n * (elem + codec.coef_bytes) / (ku["dwt_fwd_l1"] * 1e-6) / 1e9
        out["dwt_fwd_l1_frac"] = round(a / peak, 3)
        t_all = ku["dwt_fwd_l1"] + ku.get("dwt_fwd", 0.0) * cnt.get("dwt_fwd", 0)
        out["dwt_fwd_all_levels_frac"] = round(n * (elem + codec.coef_bytes) / (t_all * 1e-6) / 1e9 / peak, 3)
    if "dwt_inv_l1" in ku:
        a = n * (1 + 0.75 * s_det + elem) / (ku["dwt_inv_l1"] * 1e-6) / 1e9
        out["dwt_inv_l1_frac"] = round(a / peak, 3)
        t_all = ku["dwt_inv_l1"] + ku.get("dwt_inv", 0.0) * cnt.get("dwt_inv", 0)
        out["dwt_inv_all_levels_frac"] = round(n * (s_det + elem) / (t_all * 1e-6) / 1e9 / peak, 3)
    return out, codec


def kernel_counts(fn):
    """Launches per call of each profiled kernel name."""
    _lib.profile_enable(True)
    fn()
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    _lib.profile_enable(False)
    return {k: n for k, (ms, n) in prof.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--only", default="1,2,3,5")
    args = ap.parse_args()
    only = set(args.only.split(","))
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        peak = 6650.0
    res = {"hbm_peak_gbs": peak}
    if "1" in only:
        x = torch.from_numpy(synth.cfg1_gray12(0).astype(np.uint16)).cuda()
        x = x.unsqueeze(0).repeat(64, 1, 1, 1).contiguous()
        res["cfg1"], _ = codec_case("cfg1", x, 512, 512, 1, 12, 3, False, "chw", args.iters, peak)
    if "2" in only:
        x = torch.stack([torch.from_numpy(synth.cfg2_pathology(1000 + i)) for i in range(8)]).cuda()
        res["cfg2"], _ = codec_case("cfg2", x, 2048, 2048, 3, 8, 4, True, "hwc", args.iters, peak)
    if "3" in only or "4" in only:
        tiles = [synth.cfg2_pathology(i, 4096, 4096) for i in range(2)]
    if "3" in only:
        img = tiles[0]
        x = torch.from_numpy(img).cuda().unsqueeze(0)
        r, codec = codec_case("cfg3", x, 4096, 4096, 3, 8, 5, True, "hwc", args.iters, peak)
        cont = codec.containers[: int(codec.offsets[1])]
        hdr = ContainerHeader(4096, 4096, 3, 8, 1, 5)
        ref = x[0].to(torch.float64)
        for n in (2, 4):
            tt = timed(lambda: P.truncate_tensor(cont, hdr, n), args.iters)
            tc = P.truncate_tensor(cont, hdr, n)
            td = timed(lambda: P.decode_tensor(tc, hdr, out_dtype="int32", layout="hwc"), args.iters)
            dec = P.decode_tensor(tc, hdr, out_dtype="int32", layout="hwc").to(torch.float64)
            mse = float(((dec - ref) ** 2).mean())
            r[f"lossy_n{n}"] = {"truncate_ms": round(tt, 3), "decode_ms": round(td, 3),
                                "decode_mps": round(16.777216 / td * 1e3, 1), "bytes": int(tc.numel()),
                                "psnr_db": round(10 * np.log10(255.0 ** 2 / mse), 2) if mse > 0 else None}
        res["cfg3"] = r
        del codec
    if "4" in only:
        x = torch.stack([torch.from_numpy(tiles[i % 2]) for i in range(8)]).cuda()
        r, _ = codec_case("cfg4", x, 4096, 4096, 3, 8, 6, True, "hwc", args.iters, peak)
        r["note"] = ("8 tiles per pass (2 distinct seeded tiles repeated); a 65536^2 slide is 256 such tiles, "
                     "partitioned 256/N per GPU with no data-path collective")
        r["slide_seconds_1gpu_roundtrip"] = round(256 * 16.777216 / r["roundtrip_mps"], 3)
        res["cfg4"] = r
    if "5" in only:
        img = synth.cfg5_fluorescence(0)
        x = torch.from_numpy(img).cuda().unsqueeze(0)
        codec = Codec(8192, 8192, 4, 16, 5, False, torch.uint16, "chw", batch=1)
        codec.roundtrip_device(x)
        codec.check()
        assert torch.equal(codec.pixels_out, x)
        td = timed(lambda: codec.decode_device(), args.iters)
        ku = kernel_us(lambda: codec.decode_device(), args.iters)
        n = 4 * 8192 * 8192
        r = {"decode_ms": round(td, 3), "decode_mps": round(67.108864 / td * 1e3, 1),
             "container_bytes": int(codec.offsets[1]), "kernel_us": ku}
        if "dwt_inv_l1" in ku:  # 16-bit samples: detail depth > 16, int32 detail planes
            r["dwt_inv_l1_frac"] = round(n * (4 + 2) / (ku["dwt_inv_l1"] * 1e-6) / 1e9 / peak, 3)
            cnt = kernel_counts(lambda: codec.decode_device())
            t_all = ku["dwt_inv_l1"] + ku.get("dwt_inv", 0.0) * cnt.get("dwt_inv", 0)
            r["dwt_inv_all_levels_frac"] = round(n * (4 + 2) / (t_all * 1e-6) / 1e9 / peak, 3)
        res["cfg5"] = r
    print(json.dumps(res))


if __name__ == "__main__":
    main()
