"""Summarise an ncu --set full report of the fused query kernel into text
(key throughput metrics, stall reasons, SASS opcode histogram per query,
hottest source lines) for profiles/.

usage: ncu_summary.py REPORT.ncu-rep N_QUERIES [CUBIN KERNEL_SUBSTR] > profiles/<name>.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "smsp__cycles_active.avg",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.per_cycle_active",
    "sm__inst_executed.sum", "smsp__inst_executed.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, nq = sys.argv[1], float(sys.argv[2])
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, unit, val = raw[0], raw[1], raw[2]
    print(f"# ncu summary: {rep.split('/')[-1]}  ({int(nq)} queries per launch)")
    print(f"kernel: {val[hdr.index('Kernel Name')]}")
    print("\n## key metrics")
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k:90s} {val[i]:>16s} {unit[i]}")
    stalls = []
    for i, n in enumerate(hdr):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(val[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("\n## warp stall reasons (warps stalled per issued instruction)")
    for v, n in sorted(stalls, reverse=True)[:12]:
        print(f"{n:32s} {v:8.3f}")

    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    h, d = src[1], src[2:]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    ops = collections.Counter()
    for r in d:
        t = r[iS].strip().split()
        if not t:
            continue
        o = t[1] if t[0].startswith("@") else t[0]
        ops[o.split(".")[0]] += int(r[iE] or 0)
    tot = sum(ops.values())
    print(f"\n## SASS opcode histogram (thread-instructions per query; total {tot * 32 / nq:.1f})")
    for k, v in ops.most_common(32):
        print(f"{k:12s} {v * 32 / nq:8.1f}")

    if len(sys.argv) > 4:
        cubin, kname = sys.argv[3], sys.argv[4]
        res = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "sass_lines.py"), rep,
                              cubin, kname, str(int(nq))], capture_output=True, text=True)
        print("\n## hottest source lines (thread-instructions per query, stall samples)")
        print(res.stdout)


if __name__ == "__main__":
    main()
