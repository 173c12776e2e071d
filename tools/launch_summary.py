"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel.
usage: launch_summary.py CSV [--by-kernel]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d['Kernel Name'].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')
        if '--by-kernel' not in sys.argv:
            name = name + (' ' + d['Grid Size'] if 'gemm' in name else '')
        agg.setdefault(name, []).append(float(d['Metric Value'].replace(',', '')) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print("%-60s n=%4d  sum %9.1f us  mean %7.1f  (%4.1f%%)  first %s" % (
        k[:60], len(v), sum(v), sum(v) / len(v), 100 * sum(v) / tot, [round(x, 1) for x in v[:3]]))
print("total %.1f us" % tot)
