"""Top CUDA source lines by one ncu stall reason (per-SASS samples mapped to
lines via nvdisasm -g).  usage: stall_lines.py REPORT CUBIN KERNEL_SUBSTR REASON [n]
REASON: a source-page column such as stall_long_sb, stall_barrier, stall_wait."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname, reason = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, data = rows[1], rows[2:]
iA, iR, iS = hdr.index("Address"), hdr.index(reason), hdr.index("Source")
base = int(data[0][iA], 16)
cnt = {int(r[iA], 16) - base: (int(r[iR] or 0), r[iS].strip()) for r in data}
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
out = collections.Counter()
ops = collections.defaultdict(collections.Counter)
infn, line = False, None
for l in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        infn = kname in m.group(1)
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and line and int(m.group(1), 16) in cnt:
        v, s = cnt[int(m.group(1), 16)]
        out[line] += v
        if v:
            t = s.split()
            ops[line][(t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]] += v
tot = sum(out.values())
print(f"{reason}: {tot} samples")
for (f, ln), v in out.most_common(top):
    print(f"{v:6d} {100 * v / max(tot, 1):5.1f}%  {f}:{ln}  {dict(ops[(f, ln)].most_common(3))}")
