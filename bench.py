"""Benchmark: encode & decode megapixels/s of the B200 codec (BASELINE.json metric).

Workload (N=1, BASELINE configs[1]): 2048x2048 RGB 8-bit pathology-like images (seeded
synthetic generator, paper_2005_08713_b200/synth.py), reversible colour transform, 4 wavelet
levels, lossless.  One step = encode + decode (round trip) of `--images` such images resident
in HBM (uint8 HWC in, container bytes, uint8 HWC out), replayed as one CUDA graph.  L2 (126 MB)
is flushed by writing a 256 MB buffer between timed steps (outside the timed region).

value      whole-job MP/s = N * images * W * H / (max-over-ranks device time per step); the step
           runs as --streams concurrent sub-batches (CodecGroup)
e2e        same metric through the host-buffer API (HostPipeline.stream: K consecutive steps,
           each with pinned H2D of its pixels, encode, D2H of its container bytes, H2D of those
           host bytes, decode, D2H of its pixels; chunks on prioritised streams, batches
           overlapping across step boundaries); wall clock / K, median of 3, max over ranks.
           The isolated single-step round trip (HostPipeline.roundtrip) is reported beside it.
roofline   dominant kernel of the step, algorithmic bytes / its CUDA-event-timed duration
cpu_baseline / --impl reference: the CPU oracle port (oracle/wbpc_oracle.c) on this host

Multi-GPU (torchrun): every rank encodes/decodes its own images (tiles of a larger slide; weak
scaling) and the ranks all-gather the per-image container byte counts (NCCL) to place the
containers in one archive -- the only exchange the path has.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W = H = 2048
C = 3
BD = 8
LEVELS = 4
MP_PER_IMAGE = W * H / 1e6
METRIC = "encode & decode megapixels/s (1/2/4/8 B200) + % HBM roofline vs CPU oracle"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _gen_images(n, seed0=0):
    from paper_2005_08713_b200 import synth
    import numpy as np
    return np.stack([synth.cfg2_pathology(seed0 + i, H, W) for i in range(n)])


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"wbpc_clocks_{os.getpid()}.csv")

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sms.append(float(p[1]))
                    mx = float(p[2])
                except ValueError:
                    continue
                for nm, v in zip(names, p[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except FileNotFoundError:
            pass
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


def cpu_oracle_roundtrip(img_hwc, threads):
    """One lossless encode + decode of one cfg2 image with the C oracle; returns seconds."""
    import numpy as np
    import oracle
    from paper_2005_08713_b200 import synth
    planar = synth.planar(img_hwc).astype(np.int64)
    t = time.perf_counter()
    data = oracle.encode_image(planar, BD, LEVELS, True, threads=threads)
    dec, _ = oracle.decode_image(data, threads=threads)
    dt = time.perf_counter() - t
    assert np.array_equal(dec, planar)
    return dt, len(data)


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    imgs = _gen_images(1)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_oracle_roundtrip(imgs[0], threads)
    times = []
    for _ in range(args.steps):
        dt, _ = cpu_oracle_roundtrip(imgs[0], threads)
        times.append(dt)
    tot = sum(times)
    value = args.steps * MP_PER_IMAGE / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": "cfg2: 2048x2048 RGB8 pathology synthetic, RCT, L4, lossless encode+decode",
                   "images_per_step": 1},
        "cpu_baseline": {"value": value, "unit": "MP/s", "cores": threads, "kind": "port",
                         "sample": "1 cfg2 image (4.19 MP) encode+decode per step, oracle/wbpc_oracle.c, "
                                   f"{threads} threads over blocks"},
        "e2e": {"value": value, "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2005_08713_b200 import _lib
    from paper_2005_08713_b200.container import Codec, CodecGroup

    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B = args.images
    imgs = _gen_images(B, seed0=1000 * rank)
    x = torch.from_numpy(imgs).cuda()
    # sub-batches on concurrent streams (CodecGroup): one sequence's idle SM capacity is filled
    # by the others'; --streams 1 is the single launch sequence
    ns = args.streams if B % args.streams == 0 else 1
    codec = CodecGroup(W, H, C, BD, LEVELS, True, torch.uint8, "hwc", batch=B, streams=ns)
    sizes_local = torch.empty(B, dtype=torch.int64, device="cuda")
    sizes_all = torch.empty(B * ws, dtype=torch.int64, device="cuda")

    def step():
        codec.roundtrip_device(x)
        codec.sizes_into(sizes_local)

    # warm-up (also sets kernel attributes), correctness check
    for _ in range(2):
        step()
    codec.check()
    assert torch.equal(codec.pixels_out, x), "round trip mismatch"
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph):
            step()
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def gstep():
        graph.replay()
        if ws > 1:
            dist.all_gather_into_tensor(sizes_all, sizes_local)

    for _ in range(args.warmup):
        gstep()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 255)  # L2 flush, outside the timed events
            ev[i][0].record()
            gstep()
            ev[i][1].record()
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(tot_ms, op=dist.ReduceOp.MAX)
    tot_ms = float(tot_ms.item())
    ms_per_step = tot_ms / args.steps
    value = ws * B * MP_PER_IMAGE / (ms_per_step / 1e3)
    codec.check()
    assert torch.equal(codec.pixels_out, x), "round trip mismatch after timing"

    # ---- per-kernel breakdown with CUDA events on the launching stream (separate pass) ----
    # kernel durations from a single-stream session of the same batch (with concurrent
    # sub-batches the per-stream event intervals would overlap)
    pcodec = Codec(W, H, C, BD, LEVELS, True, torch.uint8, "hwc", batch=B)
    pcodec.roundtrip_device(x)
    pcodec.check()
    _lib.profile_enable(True)
    for i in range(args.steps):
        flush.fill_(i & 255)
        pcodec.roundtrip_device(x)
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    _lib.profile_enable(False)
    kern = {k: (ms / n * 1e3, n // args.steps) for k, (ms, n) in prof.items()}  # us per launch, launches/step
    launches = sum(n for _, n in kern.values())

    sizes = codec.container_sizes()
    enc_cb = pcodec.coef_bytes
    del pcodec
    cont_bytes = sum(sizes)
    raw_bytes = B * W * H * C
    coef_bytes = B * W * H * C * 4                 # decode side: int32 coefficients
    enc_coef_bytes = B * W * H * C * enc_cb  # encode side: int16 when the static bound allows
    peak, peak_kind = _peaks()
    per_step_us = {k: v[0] * v[1] for k, v in kern.items()}
    dom = max(per_step_us, key=per_step_us.get)
    # algorithmic bytes per launch
    alg = {
        "dwt_fwd_l1": raw_bytes + enc_coef_bytes,      # pixels in, 4 level-1 subbands out
        "dwt_inv_l1": coef_bytes + raw_bytes,          # 4 subbands in (int32), pixels out
        "block_analyze": enc_coef_bytes,               # every coefficient read once
        "block_emit": cont_bytes,                      # container bytes written
        "block_decode": cont_bytes,                    # container bytes read
        "block_reconstruct": coef_bytes,               # coefficients written
    }
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(dom)
    except Exception:  # noqa: BLE001
        pass

    def roof(name):
        us = kern[name][0]
        a = alg.get(name, 0) / (us * 1e-6) / 1e9
        return {"bound": "hbm", "achieved": round(a, 1), "peak": peak, "unit": "GB/s", "frac": round(a / peak, 4),
                "kernel": name, "us_per_launch": round(us, 1), "algorithmic_bytes_per_launch": alg.get(name, 0),
                "peak_kind": peak_kind}

    roofline = roof(dom)
    roofline["traffic"] = traffic
    dwt_roof = {k: roof(k) for k in ("dwt_fwd_l1", "dwt_inv_l1") if k in kern}

    # ---- single-image latency (B=1, no graph) ----
    codec1 = Codec(W, H, C, BD, LEVELS, True, torch.uint8, "hwc", batch=1)
    x1 = x[:1].contiguous()
    for _ in range(3):
        codec1.roundtrip_device(x1)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    enc_ms, dec_ms = [], []
    for i in range(5):
        flush.fill_(i)
        e0.record()
        codec1.encode_device(x1)
        e1.record()
        codec1.decode_device()
        e2.record()
        torch.cuda.synchronize()
        enc_ms.append(e0.elapsed_time(e1))
        dec_ms.append(e1.elapsed_time(e2))
    codec1.check()

    # ---- e2e through the host-buffer API (pipelined: chunks on separate streams) ----
    # HostPipeline.stream: K consecutive steps, each with its own pinned input -> container ->
    # pinned output round trip (every step's H2D pixels, D2H + H2D container bytes and D2H
    # pixels inside the timed region); batches overlap across step boundaries as a streaming
    # deployment would run them.  The isolated single-step round trip is reported beside it.
    from paper_2005_08713_b200.container import HostPipeline
    host = x.cpu().pin_memory()
    pipe = HostPipeline(W, H, C, BD, LEVELS, True, torch.uint8, "hwc", batch=B, chunk=max(1, B // args.e2e_chunks))
    K = max(3, min(args.steps, 6))
    outs_h = [torch.empty_like(host, pin_memory=True) for _ in range(K)]
    pipe.stream([host] * K, outs_h)
    e2e_t = []
    for i in range(3):
        flush.fill_(i)
        torch.cuda.synchronize()
        t = time.perf_counter()
        parts_all = pipe.stream([host] * K, outs_h)
        torch.cuda.synchronize()
        e2e_t.append((time.perf_counter() - t) / K)
    for o in outs_h:
        assert torch.equal(o, host), "e2e stream round trip mismatch"
    parts = parts_all[-1]
    cbytes = sum(p[0].numel() for p in parts)
    h2d = host.numel() + cbytes + sum(p[1].numel() * 8 for p in parts)
    d2h = cbytes + host.numel() + sum(p[1].numel() * 8 for p in parts)
    e2e_s = torch.tensor([statistics.median(e2e_t)], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_val = ws * B * MP_PER_IMAGE / float(e2e_s.item())
    iso_t = []
    for i in range(max(3, min(args.steps, 10))):
        flush.fill_(i)
        torch.cuda.synchronize()
        t = time.perf_counter()
        _, outs = pipe.roundtrip(host)
        torch.cuda.synchronize()
        iso_t.append(time.perf_counter() - t)
    assert torch.equal(torch.cat([o for o in outs]), host)
    iso_s = torch.tensor([statistics.median(iso_t)], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(iso_s, op=dist.ReduceOp.MAX)
    e2e_iso = ws * B * MP_PER_IMAGE / float(iso_s.item())

    cpu = None
    if rank == 0 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        dt, _ = cpu_oracle_roundtrip(imgs[0], threads)
        cpu = {"value": MP_PER_IMAGE / dt, "unit": "MP/s", "cores": threads, "kind": "port",
               "sample": f"1 cfg2 image (4.19 MP) encode+decode, oracle/wbpc_oracle.c, {threads} threads"}

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "MP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": "cfg2: 2048x2048 RGB8 pathology synthetic (seeded), RCT, L4, lossless encode+decode",
                   "images_per_step_per_gpu": B, "global_batch": B * ws, "width": W, "height": H, "channels": C,
                   "bit_depth": BD, "levels": LEVELS, "use_rct": True, "parallelism": f"tiles over {ws} GPU(s)",
                   "l2": "flushed (256 MB write) between timed steps", "cuda_graph": True,
                   "concurrent_sub_batches": ns},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_val, 1), "unit": "MP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "mode": f"HostPipeline.stream of {K} consecutive steps (wall clock / {K})",
                "isolated_step_value": round(e2e_iso, 1)},
        "gpu_launches": int(launches * ns * args.steps),  # each sub-batch runs the full sequence
        "clocks": clk.summary(),
        "encode_ms_single_image": round(statistics.median(enc_ms), 4),
        "decode_ms_single_image": round(statistics.median(dec_ms), 4),
        "dwt_roofline": dwt_roof,
        "kernel_us_per_step": {k: round(v, 1) for k, v in sorted(per_step_us.items(), key=lambda kv: -kv[1])},
        "container_bytes_per_image": round(cont_bytes / B),
        "compression_ratio": round(raw_bytes / cont_bytes, 4),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--images", type=int, default=8, help="cfg2 images per step per GPU")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--streams", type=int, default=4, help="concurrent sub-batches of the step (CodecGroup)")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="pipelined chunks of the e2e host-buffer leg")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
