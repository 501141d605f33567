"""Top source lines of an ncu report by warp-stall samples (needs -lineinfo builds).

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kn = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep] + (["--kernel-name", "regex:" + kn, "--launch-count", "1"] if kn else []) + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr, lines = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        continue
    if hdr and r[0].strip().isdigit():
        try:
            lines.append((int(r[si] or 0), int(r[ie] or 0), f"{cur_file}:{r[0]}", r[1].strip()[:70]))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in lines) or 1
print(f"total stall samples {tot}")
for s, ie_, loc, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  inst {ie_:>12d}  {loc:24s} {src}")
