"""Aggregate an ncu --set full report's per-SASS-instruction metrics (stall
samples, executed instructions) by CUDA source line, using the line table
of the kernel's cubin (built with -lineinfo).

usage: hot_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTR [TOP]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


# NMQ_HL_OUTER=<file>: attribute inlined code to its call site when the
# innermost line is not in <file> (one inlining level, nvdisasm -gi)
OUTER = os.environ.get("NMQ_HL_OUTER")


def _short(loc):
    loc = re.sub(r'^"/root/repo/paper_2305_02678_b200/csrc/', "", loc).replace('", line ', ":")
    return re.sub(r'^".*/include/', "", loc)


def line_table(lib, key):
    """SASS offset -> source line.  With OUTER set, nvdisasm -gi prints the
    inlining chain (innermost first); the innermost frame matching OUTER is
    used, suffixed with its nearest nmq_fast.cu caller."""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    table = {}
    for f in os.listdir(tmp):
        dis = subprocess.run(["nvdisasm", "-gi" if OUTER else "-g", os.path.join(tmp, f)],
                             capture_output=True, text=True).stdout
        fn, loc, chain, fresh = None, None, [], False
        for l in dis.split("\n"):
            m = re.match(r"\s*\.text\.(\S+):", l)
            if m:
                fn = m.group(1)
            if "//## File" in l:
                if not fresh:
                    chain, fresh = [], True
                chain.append(_short(l.split("//## File")[1].strip().split(" inlined at ")[0]))
                continue
            if fresh:
                fresh = False
                if OUTER:
                    hit = [i for i, c in enumerate(chain) if re.search(OUTER, c)]
                    i = hit[0] if hit else len(chain) - 1
                    loc = chain[i]
                    up = [c for c in chain[i + 1:] if c.startswith("nmq_fast.cu") and c != loc]
                    if up and not loc.startswith("nmq_fast.cu"):
                        loc += " < " + up[0]
                else:
                    loc = chain[-1]
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
            if m and fn and key in fn:
                table[int(m.group(1), 16)] = loc
    return table


def main():
    rep, lib, key = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    table = line_table(lib, key)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, iss, ie = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    tot = [0.0, 0.0]
    base = None
    for r in rows[2:]:
        try:
            a = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        base = a if base is None else base
        a -= base  # ncu reports absolute addresses; the line table is per function
        s, e = float(r[iss] or 0), float(r[ie] or 0)
        loc = table.get(a, "?")
        agg[loc][0] += s
        agg[loc][1] += e
        tot[0] += s
        tot[1] += e
    print(f"{'source line':50s} {'stall%':>7s} {'inst%':>7s}")
    for loc, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{str(loc)[:50]:50s} {100 * s / tot[0]:7.2f} {100 * e / tot[1]:7.2f}")


if __name__ == "__main__":
    main()
