"""Summarise an ncu report's source page per CUDA source line (stall samples, instructions)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kf = sys.argv[3:] and ["-k", sys.argv[3]] or []
txt = subprocess.run(["ncu", "-i", rep] + kf + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
path = None
lines = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("", "Function Name") and len(r) == len(hdr):
        lines.append((path, r))
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_ie = hdr.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[i_s] or 0) for _, r in lines) or 1
tot_ie = sum(float(r[i_ie] or 0) for _, r in lines) or 1
print(f"total samples {tot:.0f}, warp instructions {tot_ie:.0f}")
for p, r in sorted(lines, key=lambda x: -float(x[1][i_s] or 0))[:top]:
    st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
    sts = " ".join(f"{n}={v/max(float(r[i_s]),1)*100:.0f}%" for v, n in st if v)
    print(f"{float(r[i_s])/tot*100:5.1f}% ie={float(r[i_ie])/tot_ie*100:5.1f}% {p}:{r[0]:>4} {r[1].strip()[:90]:90s} {sts}")
