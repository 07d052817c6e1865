"""Per-source-line hotspot table from an ncu report (--page source, cuda,sass).
usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
files = {}
cur = None
rows = []
for line in txt.splitlines():
    if line.startswith('"File Path"'):
        cur = next(csv.reader([line]))[1]
        continue
    if line.startswith('"Line No"'):
        hdr = next(csv.reader([line]))
        continue
    if line.startswith('"Function Name"') or not line.startswith('"'):
        continue
    r = next(csv.reader([line]))
    if r[0] and r[0] != "":
        rows.append((cur, hdr, r))
out = []
for f, hdr, r in rows:
    d = dict(zip(hdr[4:], r[4:]))
    def g(k):
        try:
            return float(d.get(k, 0) or 0)
        except ValueError:
            return 0.0
    out.append((g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"), g("L1 Wavefronts Shared"),
                f.split("/")[-1], r[0], r[1][:70]))
tot = sum(o[0] for o in out) or 1
totw = sum(o[2] for o in out) or 1
toti = sum(o[1] for o in out) or 1
print(f"samples {tot:.0f}  warp-instr {toti:.3g}  smem wavefronts {totw:.3g}")
for s, i, w, f, ln, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{100*s/tot:5.1f}% stall  {100*i/toti:5.1f}% inst  {100*w/totw:5.1f}% wf  {f}:{ln:5s} {src}")
