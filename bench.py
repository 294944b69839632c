"""Benchmark: encode & decode megapixels/s of the B200 codec (BASELINE.json metric) on cfg4.

Workload (BASELINE configs[3]): the 65536^2 RGB 8-bit whole slide as 256 distinct seeded 4096^2
tiles (tile t = seed + t, the cfg2 pathology recipe, generated on the GPU: synth.cfg4_tile_torch),
6 wavelet levels, reversible colour transform, lossless; every tile is an independent container
(the reference's encode_image per tile).  The tiles are sharded contiguously over the ranks
(strong scaling: the slide is fixed, each of N GPUs holds 256/N tiles).

One step = the whole slide's round trip, device resident (SlideCodec.roundtrip_device): per batch
of tiles on its stream, encode -> rank-local archive offsets -> assembly into the rank's archive
range -> decode from the archive (batches on 4 concurrent streams, so one batch's decode overlaps
the next batches' encodes); then the all-gather of the per-tile container sizes (NCCL over NVLink
when N > 1, the path's only collective) and the archive header/index.  The inputs
(12.9 GB) exceed L2 (126 MB) many times over; L2 is also flushed (256 MB write) between steps.

value      whole-job MP/s = 65536^2 / 1e6 / (max-over-ranks device time per step)
encode_mps / decode_mps   separate encode-only (encode + exchange + assembly) and decode-only
           passes over the same slide, max over ranks
e2e        SlideCodec.roundtrip_host: pinned host tiles -> H2D -> encode -> size exchange -> D2H of
           the containers into one host archive (shared by the ranks through /dev/shm) -> H2D of
           those host bytes -> decode -> D2H of the pixels; wall clock per step, max over ranks
roofline   dominant kernel of the step: algorithmic bytes / its CUDA-event-timed duration
cpu_baseline / --impl reference: the UNMODIFIED reference (baseline/_ref, pip --target install of
           /root/reference/pkg) timed on this host's cores: one worker process per core, each
           running encode_image + decode_image (threads=1) on its own 2048^2 quarter-tile sample of
           the same generator, L6, RCT; step = one wave over all workers.

`python bench.py --gpus N` re-executes itself under torch.distributed.run with N ranks when it is
not already running under a launcher.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")

TILES_X = TILES_Y = 16
TILE = 4096
C = 3
BD = 8
LEVELS = 6
SEED = 0
METRIC = "encode & decode megapixels/s (1/2/4/8 B200) + % HBM roofline vs CPU oracle"
SAMPLE = 2048  # CPU reference sample edge (a quarter tile)


def workload_config(n_tiles: int, world: int) -> dict:
    return {"workload": f"cfg4: {TILES_X * TILE}x{TILES_Y * TILE} RGB8 whole slide as {n_tiles} distinct seeded "
                        f"{TILE}x{TILE} tiles (seed + tile index), RCT, L{LEVELS}, lossless encode+decode",
            "tiles": n_tiles, "tile": [TILE, TILE], "channels": C, "bit_depth": BD, "levels": LEVELS,
            "use_rct": True, "parallelism": f"tiles sharded contiguously over {world} GPU(s)",
            "l2": "inputs 12.9 GB >> L2; L2 also flushed (256 MB write) between timed steps"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def _dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


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


# ============================================================================ CPU reference
def _load_synth():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_wbpc_synth", os.path.join(ROOT, "paper_2005_08713_b200", "synth.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _ref_worker(conn, ref_path: str) -> None:
    """One host core: the unmodified reference's encode_image + decode_image (threads=1)."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/wbpc_numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, ref_path)
    import numpy as np
    import wbpc  # the reference package (baseline/_ref)
    synth = _load_synth()
    warm = wbpc.RasterImage.from_planes(list(np.arange(3 * 64 * 64).reshape(3, 64, 64) % 256), 8)
    wbpc.decode_image(wbpc.encode_image(warm, levels=2, use_rct=True))  # numba JIT outside timing
    conn.send(("warm", wbpc.__file__))
    while True:
        msg = conn.recv()
        if msg is None:
            break
        seed, edge = msg
        planar = synth.planar(synth.cfg2_pathology(seed, edge, edge)).astype(np.int64)
        img = wbpc.RasterImage.from_planes(list(planar), BD)
        conn.send("ready")
        conn.recv()  # go
        t0 = time.perf_counter()
        data = wbpc.encode_image(img, levels=LEVELS, use_rct=True, threads=1)
        t1 = time.perf_counter()
        dec = wbpc.decode_image(data)
        t2 = time.perf_counter()
        conn.send((t1 - t0, t2 - t1, len(data), hashlib.sha256(data).hexdigest(),
                   bool(np.array_equal(dec.samples, planar))))


class RefPool:
    """One worker process per host core running the unmodified reference; waves are timed."""

    def __init__(self, n: int | None = None):
        import multiprocessing as mp
        if not os.path.isdir(os.path.join(REF_INSTALL, "wbpc")):
            raise RuntimeError("baseline/_ref missing (pip install --target baseline/_ref the reference)")
        cores = len(os.sched_getaffinity(0))
        try:  # ~2 GB peak per worker at 2048^2
            import psutil
            cores = max(1, min(cores, int(psutil.virtual_memory().available / 2.5e9)))
        except Exception:  # noqa: BLE001
            pass
        self.n = n or cores
        ctx = mp.get_context("spawn")
        self.conns, self.procs = [], []
        for _ in range(self.n):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_ref_worker, args=(b, REF_INSTALL), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        self.ref_file = [c.recv() for c in self.conns][0][1]

    def wave(self, seeds, edge=SAMPLE):
        for c, s in zip(self.conns, seeds):
            c.send((s, edge))
        for c in self.conns[:len(seeds)]:
            assert c.recv() == "ready"
        t0 = time.perf_counter()
        for c in self.conns[:len(seeds)]:
            c.send("go")
        res = [c.recv() for c in self.conns[:len(seeds)]]
        wall = time.perf_counter() - t0
        assert all(r[4] for r in res), "reference round trip not lossless"
        return wall, res

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:  # noqa: BLE001
                pass
        for p in self.procs:
            p.join(timeout=10)


def _sample_seed(step: int, k: int) -> int:
    return SEED + 100000 + 64 * step + k


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    try:
        pool = RefPool(args.ref_workers or None)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"reference not installed in baseline/_ref: {e!r}"}),
              flush=True)
        return 0
    mp_sample = SAMPLE * SAMPLE / 1e6
    walls = []
    try:
        for i in range(args.warmup + args.steps):
            wall, res = pool.wave([_sample_seed(i, k) for k in range(pool.n)])
            if i >= args.warmup:
                walls.append(wall)
    finally:
        pool.close()
    tot = sum(walls)
    value = args.steps * pool.n * mp_sample / tot
    sample = (f"per step, {pool.n} worker processes (one per host core) each run the unmodified reference "
              f"(baseline/_ref {os.path.relpath(pool.ref_file, ROOT)}) encode_image + decode_image, threads=1, on "
              f"its own {SAMPLE}x{SAMPLE} quarter-tile sample of the cfg4 generator (numpy, distinct seeds), L{LEVELS}, "
              f"RCT; numba JIT warmed outside timing; step time = wave wall clock")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "MP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": workload_config(args.tiles, ws),
        "cpu_baseline": {"value": round(value, 4), "unit": "MP/s", "cores": pool.n, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(gpu_encode_sha):
    """Rank 0, N=1: one wave of the reference over all host cores + single-thread figures.

    gpu_encode_sha(planar uint8 (C,H,W)) -> sha256 of this repo's GPU container for the sample,
    checked against the reference's bytes for sample 0.
    """
    import numpy as np
    pool = RefPool()
    try:
        seeds = [_sample_seed(0, k) for k in range(pool.n)]
        wall, res = pool.wave(seeds)
    finally:
        pool.close()
    mp_sample = SAMPLE * SAMPLE / 1e6
    single = [r[0] + r[1] for r in res]
    synth = _load_synth()
    planar = synth.planar(synth.cfg2_pathology(seeds[0], SAMPLE, SAMPLE))
    match = gpu_encode_sha(planar) == res[0][3]
    port = None
    try:
        import oracle  # the C restatement, CPU-baseline leg only
        oracle.build()
        t = time.perf_counter()
        data = oracle.encode_image(planar.astype(np.int64), BD, LEVELS, True, threads=1)
        oracle.decode_image(data, threads=1)
        port = {"value": round(mp_sample / (time.perf_counter() - t), 4), "unit": "MP/s", "cores": 1, "kind": "port",
                "sample": f"sample 0, oracle/wbpc_oracle.c (C restatement), 1 thread"}
    except Exception as e:  # noqa: BLE001
        port = {"unavailable": repr(e)}
    return {"value": round(pool.n * mp_sample / wall, 4), "unit": "MP/s", "cores": pool.n, "kind": "reference",
            "sample": (f"one wave: {pool.n} worker processes (one per core), each the unmodified reference "
                       f"(baseline/_ref) encode_image + decode_image (threads=1) of its own {SAMPLE}x{SAMPLE} "
                       f"quarter-tile sample, L{LEVELS}, RCT; wall {wall:.2f} s"),
            "single_thread": {"value": round(mp_sample / statistics.median(single), 4), "unit": "MP/s", "cores": 1,
                              "kind": "reference", "sample": "median worker of the same wave"},
            "port_single_thread": port,
            "gpu_container_bitexact_vs_reference_sample0": bool(match)}


# ============================================================================ GPU
def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2005_08713_b200 import _lib, synth
    from paper_2005_08713_b200.slide import SlideCodec, release_host_buffer, shared_host_buffer

    ws, rank, local = _dist_env()
    # WBPC_BENCH_BACKEND=gloo (with ranks sharing the visible GPUs) exercises the multi-rank path
    # on a single GPU for testing; measured runs use NCCL, one rank per GPU
    backend = os.environ.get("WBPC_BENCH_BACKEND", "nccl")
    dev_index = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(dev_index)
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init log (nranks) for the record
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries only the JSON line
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    n_tiles = args.tiles
    tx = TILES_X if n_tiles == TILES_X * TILES_Y else n_tiles
    ty = n_tiles // tx
    codec = SlideCodec(tx, ty, TILE, TILE, C, BD, LEVELS, True, torch.uint8, "hwc", world=ws, rank=rank,
                       batch=args.batch, streams=args.streams)
    nl = codec.n_local
    x = torch.empty((nl, TILE, TILE, C), dtype=torch.uint8, device="cuda")
    for i in range(nl):
        synth.cfg4_tile_torch(SEED, codec.first + i, TILE, "cuda", out=x[i])
    out = torch.empty_like(x)
    slide_mp = n_tiles * TILE * TILE / 1e6

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # first round trip: checks every tile is restored exactly
    codec.roundtrip_device(x, out)
    codec.check()
    assert torch.equal(out, x), "slide round trip mismatch"
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        codec.roundtrip_device(x, out)
    barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    with ClockSampler(dev_index) as clk:
        for i in range(args.steps):
            flush.fill_(i & 255)  # L2 flush, outside the timed events
            evs[i][0].record()
            codec.roundtrip_device(x, out)
            evs[i][1].record()
        torch.cuda.synchronize()
    barrier()
    tot = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / args.steps
    value = slide_mp / (ms_per_step / 1e3)
    codec.check()
    assert torch.equal(out, x), "slide round trip mismatch after timing"
    # encode alone (encode + size exchange + archive assembly) and decode alone (from the archive),
    # same slide, same timing rules
    out.zero_()
    ph = {"enc": [], "dec": []}
    for i in range(args.steps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        flush.fill_(i & 255)
        e[0].record()
        codec.encode(x)
        codec.exchange()
        codec.assemble()
        e[1].record()
        flush.fill_((i + 1) & 255)
        e[2].record()
        codec.decode(out)
        e3 = torch.cuda.Event(enable_timing=True)
        e3.record()
        ph["enc"].append((e[0], e[1]))
        ph["dec"].append((e[2], e3))
    torch.cuda.synchronize()
    codec.check()
    assert torch.equal(out, x), "phased round trip mismatch"
    pt = torch.tensor([sum(a.elapsed_time(b) for a, b in ph["enc"]), sum(a.elapsed_time(b) for a, b in ph["dec"])],
                      dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(pt, op=dist.ReduceOp.MAX)
    enc_ms, dec_ms = (float(v) for v in pt.tolist())
    sizes = codec.tile_sizes()
    cont_total = sum(sizes)
    cont_local = int(codec.local_off[-1].item())
    archive_total = int(codec.base_total[1].item())

    # ---- per-kernel breakdown: CUDA events on the launching stream, single-stream pass ----
    S = codec.S
    codec.S = 1
    _lib.profile_enable(True)
    prof_steps = max(1, min(args.steps, 2))
    for i in range(prof_steps):
        flush.fill_(i)
        codec.roundtrip_device(x, out)
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    _lib.profile_enable(False)
    codec.S = S
    kern = {k: (ms / n * 1e3, n // prof_steps) for k, (ms, n) in prof.items()}  # us per launch, launches/step
    launches_per_step = sum(n for _, n in kern.values())
    per_step_us = {k: v[0] * v[1] for k, v in kern.items()}
    B = codec.B
    raw_b = B * TILE * TILE * C                      # pixel bytes per batch launch
    coef_enc = raw_b * codec.coef_bytes              # encode side: int16 when the static bound allows
    # decode side: detail planes int16 when every detail block has depth <= 16, which the encoder's
    # static int16 bound implies for these containers; the level-1 LL plane the last inverse level
    # reads is int32 (a quarter of the samples)
    s_det = 2 if codec.coef_bytes == 2 else 4
    coef_dec = raw_b * s_det
    cont_b = cont_local / max(1, codec.nb)           # mean container bytes per batch launch
    alg = {
        "dwt_fwd_l1": raw_b + coef_enc,              # pixels in, the 4 level-1 subbands out
        "dwt_inv_l1": raw_b + 3 * coef_dec // 4 + raw_b,  # LL1 (int32) + 3 detail subbands in, pixels out
        "block_symbols": coef_enc,                   # every coefficient read once
        "block_emit": cont_b,                        # container bytes written
        "block_decode": cont_b,                      # container bytes read
        "block_reconstruct": coef_dec,               # coefficients written (detail width)
        "archive_gather": 2 * cont_local,            # the rank's containers read + written once
    }
    peak, peak_kind = _peaks()
    dom = max(per_step_us, key=per_step_us.get)
    traffic = None
    try:  # ncu DRAM bytes per launch of the captured batch size, scaled to this run's batch
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t4 = json.load(f).get("cfg4", {})
        if dom in t4:
            traffic = int(t4[dom] * B / t4.get("_tiles_per_launch", B))
    except Exception:  # noqa: BLE001
        pass

    def roof(name, nbytes=None, us=None):
        us = kern[name][0] if us is None else us
        nbytes = alg.get(name, 0) if nbytes is None else nbytes
        a = nbytes / (us * 1e-6) / 1e9
        return {"bound": "hbm", "achieved": round(a, 1), "peak": peak, "unit": "GB/s", "frac": round(a / peak, 4),
                "kernel": name, "us_per_launch": round(us, 1), "algorithmic_bytes_per_launch": int(nbytes),
                "peak_kind": peak_kind}

    roofline = roof(dom)
    roofline["traffic"] = traffic
    dwt = {k: roof(k) for k in ("dwt_fwd_l1", "dwt_inv_l1") if k in kern}
    # SURVEY §8(d) accounting: all levels together, compulsory bytes C*(s_in + s_coef) per pixel
    if "dwt_fwd_l1" in kern and "dwt_fwd" in per_step_us:
        us = (per_step_us["dwt_fwd_l1"] + per_step_us["dwt_fwd"]) / max(1, codec.nb)
        dwt["forward_all_levels"] = roof("dwt_fwd_l1", raw_b + coef_enc, us) | {"kernel": "dwt_fwd_l1 + dwt_fwd"}
    if "dwt_inv_l1" in kern and "dwt_inv" in per_step_us:
        us = (per_step_us["dwt_inv_l1"] + per_step_us["dwt_inv"]) / max(1, codec.nb)
        dwt["inverse_all_levels"] = roof("dwt_inv_l1", coef_dec + raw_b, us) | {"kernel": "dwt_inv_l1 + dwt_inv"}
    codec_bytes = 2 * n_tiles * TILE * TILE * C + 2 * cont_total
    whole = {"bytes_per_step": codec_bytes, "frac": round(codec_bytes / (ms_per_step / 1e3) / 1e9 / peak / ws, 4),
             "definition": "(raw in + container out + container in + raw out) / step time / (N x HBM peak)"}

    # ---- e2e: pinned host tiles -> host archive -> pinned host tiles ----
    e2e = None
    if not args.no_e2e:
        x_host = torch.empty((nl, TILE, TILE, C), dtype=torch.uint8, pin_memory=True)
        x_host.copy_(x)
        out_host = torch.empty_like(x_host, pin_memory=True)
        keep = None
        shared = False
        if ws > 1:
            # one archive shared by the ranks in /dev/shm when it has room (a short tmpfs would end
            # the ranks with SIGBUS while the pages are pinned), else a pinned archive per rank
            path = f"/dev/shm/wbpc_archive_{os.environ.get('MASTER_PORT', '0')}"
            room = torch.zeros(1, dtype=torch.int32, device="cuda")
            if rank == 0:
                try:
                    st = os.statvfs("/dev/shm")
                    room[0] = int(st.f_bavail * st.f_frsize >= archive_total + (256 << 20))
                except OSError:
                    pass
            dist.broadcast(room, 0)
            shared = bool(room.item())
            okf = torch.ones(1, dtype=torch.int32, device="cuda")
            if shared:
                try:
                    if rank == 0:
                        arch, keep = shared_host_buffer(path, archive_total, create=True)
                    dist.barrier()
                    if rank != 0:
                        arch, keep = shared_host_buffer(path, archive_total, create=False)
                except Exception:  # noqa: BLE001
                    okf[0] = 0
                dist.all_reduce(okf, op=dist.ReduceOp.MIN)
                if not okf.item():
                    if keep is not None:
                        release_host_buffer(keep)
                        keep = None
                    shared = False
            if not shared:
                arch = torch.empty(archive_total, dtype=torch.uint8, pin_memory=True)
        else:
            arch = torch.empty(archive_total, dtype=torch.uint8, pin_memory=True)
        codec.roundtrip_host(x_host, out_host, arch)  # warm
        torch.cuda.synchronize()
        ts = []
        if ws == 1:
            # slides streamed back to back (SlideCodec.stream_host): wall clock / slides, 3 runs
            K = args.e2e_steps
            for i in range(3):
                flush.fill_(i)
                torch.cuda.synchronize()
                t = time.perf_counter()
                codec.stream_host([x_host] * K, [out_host] * K, [arch] * K)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t) / K)
        else:
            for i in range(args.e2e_steps):
                flush.fill_(i)
                barrier()
                t = time.perf_counter()
                codec.roundtrip_host(x_host, out_host, arch)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t)
        codec.check()
        assert torch.equal(out_host, x_host), "e2e round trip mismatch"
        barrier()
        # the host archive is the device archive, byte for byte (this rank's range + rank 0's index)
        base = int(codec.base_total[0].item())
        ok = torch.equal(arch[base:base + cont_local], codec.archive_dev[:cont_local].cpu())
        if rank == 0:
            ok = ok and torch.equal(arch[:codec.index.numel()], codec.index.cpu())
        med = torch.tensor([statistics.median(ts), float(not ok)], dtype=torch.float64, device="cuda")
        if ws > 1:
            dist.all_reduce(med, op=dist.ReduceOp.MAX)
        assert med[1].item() == 0, "host archive differs from the device archive"
        e2e = {"value": round(slide_mp / float(med[0]), 1), "unit": "MP/s",
               "h2d_bytes_per_step": int(n_tiles * TILE * TILE * C + cont_total),
               "d2h_bytes_per_step": int(n_tiles * TILE * TILE * C + cont_total + codec.index.numel()),
               "mode": ((f"SlideCodec.stream_host of {args.e2e_steps} slides back to back, wall clock / slides "
                         f"(median of 3 runs)" if ws == 1 else
                         f"SlideCodec.roundtrip_host per slide, wall clock (median of {args.e2e_steps}, max over "
                         f"ranks)") +
                        f": per batch H2D tiles, encode, D2H containers into the host archive "
                        f"({'/dev/shm, shared by the ranks' if shared else 'pinned'}), H2D of those host bytes, "
                        f"decode, D2H tiles; bytes are whole-job per slide")}
        del x_host, out_host
        if keep is not None:
            barrier()
            release_host_buffer(keep)
        if ws > 1 and rank == 0 and os.path.exists(path):
            os.unlink(path)

    # the reference-compatible functional API on one tile (host RasterImage -> bytes -> RasterImage,
    # int64 host samples as the reference returns them): the drop-in path's per-call figure
    dropin = None
    if rank == 0 and not args.no_e2e:
        import numpy as np
        from paper_2005_08713_b200 import RasterImage, decode_image, encode_image
        planar = x[0].permute(2, 0, 1).contiguous().cpu().numpy().astype(np.int64)
        img = RasterImage.from_planes(list(planar), BD)
        data = encode_image(img, levels=LEVELS, use_rct=True)
        back = decode_image(data)
        assert np.array_equal(back.samples, planar), "drop-in round trip mismatch"
        te, td = [], []
        for _ in range(3):
            t = time.perf_counter()
            data = encode_image(img, levels=LEVELS, use_rct=True)
            t1 = time.perf_counter()
            decode_image(data)
            te.append(t1 - t)
            td.append(time.perf_counter() - t1)
        tmp = TILE * TILE / 1e6
        dropin = {"encode_image_mps": round(tmp / statistics.median(te), 1),
                  "decode_image_mps": round(tmp / statistics.median(td), 1),
                  "roundtrip_mps": round(tmp / (statistics.median(te) + statistics.median(td)), 1),
                  "sample": "one 4096x4096 tile through encode_image / decode_image (RasterImage with int64 "
                            "host samples in and out, container bytes on the host), median of 3"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        from paper_2005_08713_b200.container import encode_tensor

        def gpu_sha(planar):
            t = torch.from_numpy(planar).cuda()
            buf, offs = encode_tensor(t, BD, LEVELS, True, "chw")
            return hashlib.sha256(buf[offs[0]:offs[1]].cpu().numpy().tobytes()).hexdigest()
        try:
            cpu = cpu_baseline(gpu_sha)
        except Exception as e:  # noqa: BLE001
            cpu = {"unavailable": repr(e)}

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "MP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(n_tiles, ws),
        "run": {"tiles_per_gpu": nl, "batch_tiles": codec.B, "concurrent_streams": codec.S,
                "step": ("per batch on its stream: encode -> rank-local archive offsets (ordered across batches) -> "
                         "archive assembly -> decode from the archive; then the size all-gather and the archive "
                         "index"),
                "encode_decode_split": "encode_mps / decode_mps from separate encode-only (encode, size "
                                       "exchange, assembly) and decode-only passes over the slide"},
        "encode_mps": round(slide_mp / (enc_ms / args.steps / 1e3), 1),
        "decode_mps": round(slide_mp / (dec_ms / args.steps / 1e3), 1),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_dropin_api": dropin,
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk.summary(),
        "whole_codec_roofline": whole,
        "dwt_roofline": dwt,
        "kernel_us_per_step": {k: round(v, 1) for k, v in sorted(per_step_us.items(), key=lambda kv: -kv[1])},
        "container_bytes_slide": int(cont_total),
        "archive_bytes": archive_total,
        "compression_ratio": round(n_tiles * TILE * TILE * C / cont_total, 4),
        "tile_sizes_sha256": hashlib.sha256(json.dumps(sizes).encode()).hexdigest(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--tiles", type=int, default=TILES_X * TILES_Y, help="tiles of the slide (256 = cfg4)")
    ap.add_argument("--batch", type=int, default=8, help="tiles per encode/decode launch sequence")
    ap.add_argument("--streams", type=int, default=4, help="concurrent batch streams per GPU")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-workers", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}", file=sys.stderr)
            return 2
    elif args.gpus > 1:
        # self-launch: one rank per GPU under torch.distributed.run (NCCL rendezvous on 127.0.0.1)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
