"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list
(tools/r02_refresh.sh over tools/prof_cmd.sh): our kernels only, totals per
kernel, and one full step of each pipeline (C5r, config 5 as written) in
launch order, taken from the second fused-K1 launch of its kind onward.

  python tools/launch_summary.py profiles/r02_launches.csv > profiles/r02_launches_summary.txt
"""
import collections
import csv
import re
import sys

OURS = ("ssb::", "seq_fill_kernel", "note_overflow_kernel", "note_capacity_kernel")


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("(int)", "").replace("(bool)", "")
    return re.sub(r"\s+", " ", name).strip()


rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = v / 1e3 if r["Metric Unit"] in ("ns", "nsecond") else v * 1e3 if r["Metric Unit"] in ("ms", "msecond") else v
    rows.append((int(r["ID"]), r["Kernel Name"], us))
ours = [(i, short(n), us) for i, n, us in rows if any(k in n for k in OURS)]
tot = collections.defaultdict(lambda: [0, 0.0])
for _, n, us in ours:
    tot[n][0] += 1
    tot[n][1] += us
total = sum(us for _, _, us in ours)
print("ncu --metrics gpu__time_duration.sum --clock-control none, tools/prof_cmd.sh; cold-cache serialised")
print(f"per-launch times; our kernels only ({len(ours)} of {len(rows)} launches: the rest are torch input synthesis)")
print(f"{len(ours)} launches, {total / 1e3:.3f} ms total")
for n, (c, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:58s} {c:3d} launches {us / 1e3:9.3f} ms {100 * us / total:5.1f}%")


def step(k1_pat: str, title: str) -> None:
    idx = [k for k, (_, n, _) in enumerate(ours) if re.search(k1_pat, n)]
    if len(idx) < 2:
        return
    a = idx[1]
    b = a + 1
    while b < len(ours) and "fft_mag_kernel" not in ours[b][1] and "psd_tile" not in ours[b][1]:
        b += 1
    seg = ours[a:b]
    t = sum(us for _, _, us in seg)
    print(f"\n{title}, in launch order (second K1 launch of its kind):")
    for _, n, us in seg:
        print(f"{us:12.1f} us {100 * us / t:5.1f}%  {n}")
    print(f"{t:12.1f} us total")


step(r"fft_mag_kernel<12, 0, 1, 0, 0>", "One C5r step (296 captures, rect)")
step(r"fft_mag_kernel<12, 0, 1, 1, 1>", "One config-5-as-written step (296 Hann plots, 4881 rows)")
