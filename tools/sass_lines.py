"""Attribute ncu per-SASS-instruction execution counts to CUDA source lines
(nvdisasm -g line info).  usage: sass_lines.py REPORT.ncu-rep CUBIN KERNEL_SUBSTR [n_queries]"""
import csv, io, re, subprocess, sys, collections
rep, cubin, kname = sys.argv[1:4]
nq = float(sys.argv[4]) if len(sys.argv) > 4 else 2073600
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                        capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(csvtxt)))
hdr = rows[1]; data = rows[2:]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][iA], 16)
cnt = {int(r[iA], 16) - base: (int(r[iE] or 0), int(r[iW] or 0), r[iS].strip()) for r in data}
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# find the kernel's section
out = collections.defaultdict(lambda: [0, 0])
cur_fn = None; line = None; infn = False
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
    if m and line:
        off = int(m.group(1), 16)
        if off in cnt:
            out[line][0] += cnt[off][0]
            out[line][1] += cnt[off][1]
tot = sum(v[0] for v in out.values())
print(f"total lane-instr/query {tot*32/nq:.1f}")
src = {}
for (f, ln), (e, w) in sorted(out.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[5]) if len(sys.argv) > 5 else 45]:
    if f not in src:
        try:
            src[f] = open(subprocess.run(["bash", "-c", f"ls paper_2305_02678_b200/csrc/{f}"], capture_output=True, text=True).stdout.strip()).read().splitlines()
        except Exception:
            src[f] = []
    txt = src[f][ln - 1].strip()[:70] if ln - 1 < len(src[f]) else ""
    print(f"{e*32/nq:7.1f} /q  stall {w:5d}  {f}:{ln:<5d} {txt}")
