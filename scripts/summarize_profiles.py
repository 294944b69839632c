"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

usage: python scripts/summarize_profiles.py <tag> <launches.csv> <full.ncu-rep> [workload key, default cfg4]
writes profiles/<tag>_launches_summary.txt, profiles/<tag>_ncu_full_summary.txt and
profiles/ncu_traffic.json (DRAM bytes per launch by bench kernel name, for bench.py's
roofline `traffic` field).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, launches, rep = sys.argv[1:4]
wkey = sys.argv[4] if len(sys.argv) > 4 else "cfg4"
PROF = os.path.join(ROOT, "profiles")

# kernel (demangled prefix) -> bench profile name
NAMES = [("k_fwd_rgb8_tma", "dwt_fwd_l1"), ("k_fwd_l1", "dwt_fwd_l1"), ("k_fwd_tile", "dwt_fwd"),
         ("k_inv_tile", "dwt_inv"), ("k_inv<3, 1", "dwt_inv_l1"), ("k_inv<1, 1", "dwt_inv_l1"),
         ("k_inv<4, 1", "dwt_inv_l1"), ("k_inv<1, 0", "dwt_inv"), ("k_inv2<3, 1", "dwt_inv_l1"),
         ("k_inv2<1, 0", "dwt_inv"), ("k_fwd_i16_tma", "dwt_fwd"), ("k_block_analyze", "block_analyze"), ("k_block_symbols", "block_symbols"),
         ("k_block_huffman", "block_huffman"), ("k_block_sizes", "block_sizes"),
         ("k_block_emit", "block_emit"), ("k_block_planes", "block_decode"), ("k_block_header", "block_header"),
         ("k_block_reconstruct", "block_reconstruct"), ("k_offsets", "offsets"), ("k_zero_out", "zero_out"),
         ("k_index_check", "index_check"), ("k_block_errors", "block_errors"), ("k_level0", "dwt_fwd"),
         ("k_gather_tiles", "archive_gather"), ("k_tile_sizes", "archive_sizes"), ("k_archive_index", "archive_index")]


def bench_name(k):
    for pre, n in NAMES:
        if k.startswith(pre) or ("wb::" + pre) in k or k.startswith("void " + pre) or ("void wb::" + pre) in k:
            return n
    return None


# ---- launch list (gpu__time_duration per launch, serialised / cold under ncu)
rows = [r for r in csv.reader(open(launches)) if r and not r[0].startswith("==")]
hdr = rows[0]
ik, iv, imn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if len(r) != len(hdr) or r[imn] != "gpu__time_duration.sum":
        continue
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    n = bench_name(r[ik]) or r[ik][:40]
    tot[n] += v
    cnt[n] += 1
unit = rows[1][hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
allt = sum(tot.values())
with open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (launch list of bench.py --steps 2"
            f" --warmup 3 --no-cpu); cold-cache serialised launches: shares, not absolute step times\n")
    f.write(f"# source: {os.path.basename(launches)}; time unit {unit}\n")
    f.write(f"{'kernel':22s} {'launches':>8s} {'total':>14s} {'share':>7s}\n")
    for n, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write(f"{n:22s} {cnt[n]:8d} {v:14.0f} {v / allt * 100:6.1f}%\n")
print(open(os.path.join(PROF, f"{tag}_launches_summary.txt")).read())

# ---- full capture: per kernel metrics
mets = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mets)],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(txt.splitlines()))
h = rr[0]
units = rr[1]
traffic = defaultdict(list)
lines = []
for r in rr[2:]:
    k = r[h.index("Kernel Name")]
    vals = {m: (r[h.index(m)], units[h.index(m)]) for m in mets}

    def num(m, scale):
        v, u = vals[m]
        v = float(v.replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
                    "msecond": 1e3, "usecond": 1, "nsecond": 1e-3}.get(u, 1) / scale
    dur_us = num("gpu__time_duration.sum", 1)
    rd, wr = num("dram__bytes_read.sum", 1), num("dram__bytes_write.sum", 1)
    n = bench_name(k) or k[:30]
    traffic[n].append(rd + wr)
    lines.append(f"{n:18s} {k[:34]:34s} {dur_us:9.1f} us  dram rd {rd/1e6:8.1f} MB wr {wr/1e6:8.1f} MB  "
                 f"({(rd+wr)/dur_us/1e3:7.1f} GB/s)  sm {float(vals[mets[3]][0]):5.1f}%  "
                 f"warps {float(vals[mets[5]][0]):5.1f}%  issue {float(vals[mets[6]][0]):5.1f}%  "
                 f"regs {vals[mets[7]][0]} grid {vals[mets[8]][0]} block {vals[mets[9]][0]}  "
                 f"warp-eff {float(vals[mets[10]][0]) / 32 * 100:5.1f}%")
with open(os.path.join(PROF, f"{tag}_ncu_full_summary.txt"), "w") as f:
    f.write(f"# ncu --set full --clock-control none (scripts/ncu_target.py NCU_CFG={wkey}: one profiled round\n"
            "# trip after a warm-up); per kernel launch.  ncu flushes caches per replay.\n"
            "# warp-eff = smsp__thread_inst_executed_per_inst_executed / 32 (warp execution efficiency)\n")
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
tpath = os.path.join(PROF, "ncu_traffic.json")
try:
    allt = json.load(open(tpath))
    if not all(isinstance(v, dict) for v in allt.values()):
        allt = {"cfg2": allt}
except Exception:  # noqa: BLE001
    allt = {}
allt[wkey] = {k: round(sum(v) / len(v)) for k, v in traffic.items() if not k.startswith(("void at::", "wb::"))}
if wkey == "cfg4":
    allt[wkey]["_tiles_per_launch"] = int(os.environ.get("NCU_TILES", "4"))
json.dump(allt, open(tpath, "w"), indent=1)
