"""Top SASS instructions by warp-stall samples from an ncu report:
python tools/ncu_sass_top.py report.ncu-rep [N] [kernel-substring]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
print("total samples", tot, "instructions", len(body))
ranked = sorted(range(len(body)), key=lambda i: -int(body[i][ix["Warp Stall Sampling (All Samples)"]] or 0))
for i in ranked[:top]:
    r = body[i]
    print("%5d %5.1f%% %8s  %-60s exec=%s" % (i, 100.0 * int(r[ix["Warp Stall Sampling (All Samples)"]]) / max(tot, 1),
                                        r[ix["Address"]][-5:], r[ix["Source"]].strip()[:60], r[ix["Instructions Executed"]]))
