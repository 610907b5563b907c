"""Summarise an ncu report (read here, no GPU): key metrics + SASS hot spots."""
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def details(rep):
    out = {}
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        out[(d.get("Section Name"), d.get("Metric Name"))] = (d.get("Metric Value"), d.get("Metric Unit"))
    return out


def raw(rep, names):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for n in names:
        for i, h in enumerate(hdr):
            if h == n:
                res[n] = (vals[i], units[i])
    return res


def hot(rep, top=25):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    groups = []
    for r in data:
        n = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        if groups and groups[-1][1] == n:
            groups[-1][2] += 1
            groups[-1][3] += s
        else:
            groups.append([r[ix["Address"]], n, 1, s, r[ix["Source"]]])
    tot = sum(g[1] * g[2] for g in groups) or 1
    ts = sum(g[3] for g in groups) or 1
    print(f"total warp instructions {tot}, stall samples {ts}")
    for g in sorted(groups, key=lambda g: -g[3])[:top]:
        print(f"{g[0][-6:]} exec {g[1]:>8} x{g[2]:>3} = {100 * g[1] * g[2] / tot:5.1f}% instr, "
              f"{100 * g[3] / ts:5.1f}% stalls  {g[4][:60]}")


if __name__ == "__main__":
    rep = sys.argv[1]
    d = details(rep)
    for k in [("GPU Speed Of Light Throughput", "Duration"), ("GPU Speed Of Light Throughput", "DRAM Throughput"),
              ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"), ("Compute Workload Analysis", "Executed Ipc Active"),
              ("Scheduler Statistics", "Issued Warp Per Scheduler"), ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
              ("Occupancy", "Achieved Active Warps Per SM"), ("Instruction Statistics", "Executed Instructions"),
              ("Launch Statistics", "Registers Per Thread"), ("Launch Statistics", "Block Size"), ("Launch Statistics", "Grid Size")]:
        print(k[1].ljust(40), d.get(k))
    r = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "smsp__average_warp_latency_issue_stalled_barrier", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                  "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__sass_average_branch_targets_threads_uniform.pct"])
    for k, v in r.items():
        print(k.ljust(60), v)
    stall = raw(rep, [])
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    st = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    st = sorted(((h, float(v or 0)) for h, v in st), key=lambda x: -x[1])[:12]
    print("stall reasons (samples):")
    for h, v in st:
        print("   ", h.replace("smsp__pcsamp_warps_issue_stalled_", "").ljust(40), v)
    hot(rep)
