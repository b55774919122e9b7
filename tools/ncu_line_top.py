"""Per CUDA source line: instructions executed and stall samples, from an
ncu report's cuda,sass source view.
python tools/ncu_line_top.py report.ncu-rep [launch-skip] [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
ex = defaultdict(int); st = defaultdict(int); src = {}
cur_file, cur_line = None, None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a CUDA source line row
        cur_line = (cur_file, int(r[0]))
        src[cur_line] = r[1].strip()[:70]
    e = r[hdr["Instructions Executed"]]
    s = r[hdr["Warp Stall Sampling (All Samples)"]]
    if cur_line and e:
        try:
            ex[cur_line] += int(e); st[cur_line] += int(s or 0)
        except ValueError:
            pass
T = sum(ex.values()); S = sum(st.values())
print("instructions", T, "stall samples", S)
for k in sorted(ex, key=lambda k: -ex[k])[:top]:
    print("%6.2f%% inst %6.2f%% stall  %s:%d  %s" % (100 * ex[k] / T, 100 * st[k] / max(S, 1), k[0], k[1], src.get(k, "")))
