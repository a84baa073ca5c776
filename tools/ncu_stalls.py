"""Top SASS lines by warp-stall samples from an ncu report (source page, sass view).

    python tools/ncu_stalls.py REP [--skip N] [--top 25]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--skip", type=int, default=0)
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--launch-skip", str(a.skip), "--launch-count",
                      "1", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out))]
hdr = next(r for r in rows if "Address" in r and "Source" in r)
data = [r for r in rows if len(r) == len(hdr) and r != hdr]
i_s, i_src, i_a = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Address")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[i_s]) for r in data) or 1.0
print(f"{len(data)} SASS lines, {tot:.0f} samples")
for r in sorted(data, key=lambda r: -f(r[i_s]))[: a.top]:
    print(f"{f(r[i_s]) / tot * 100:5.1f}%  {r[i_a]}  {r[i_src][:110]}")
