"""Map ncu SASS-level stall samples of one kernel to CUDA source lines.
usage: ncu_lines.py <report.ncu-rep> <kernel-regex> <mangled-name> <cubin> [top]"""
import collections, csv, io, re, subprocess, sys

rep, kre, mangled, cubin = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
data = rows[2:]
si, ai = h.index("Warp Stall Sampling (All Samples)"), h.index("Address")
base = min(int(r[ai], 16) for r in data)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if re.match(rf"\s*\.text\.{re.escape(mangled)}:", l))
lines, cur = {}, None
for l in dis[start + 1:]:
    if l.strip().startswith(".section") and ".text." in l:
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
agg = collections.Counter()
for r in data:
    agg[lines.get(int(r[ai], 16) - base, ("?", 0))] += float(r[si] or 0)
tot = sum(agg.values())
for (f, ln), v in agg.most_common(top):
    print(f"{v / tot:.3f}  {f}:{ln}")
