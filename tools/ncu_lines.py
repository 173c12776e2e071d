"""Aggregate ncu warp-stall samples per CUDA source line.
usage: ncu_lines.py REP KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, fname, hdr = {}, "", None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0] not in ("", "-"):
        try:
            v = float(r[4])
        except ValueError:
            continue
        key = (fname, int(r[0]))
        agg[key] = [agg.get(key, [0, ""])[0] + v, r[1][:100]]
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (v, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:N]:
    print("%5.1f%%  %s:%d  %s" % (100 * v / tot, f, ln, src.strip()))
