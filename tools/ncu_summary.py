"""Summarise an ncu report: key section metrics, stall hot spots, instruction mix.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Dynamic Shared Memory Per Block",
        "Block Limit Shared Mem", "Block Limit Registers", "Grid Size"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    out = {}
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            out[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if len(raw) >= 3:
        names, units, vals = raw[0], raw[1], raw[2]
        for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                     "smsp__inst_executed_op_shared_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                     "sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
                     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                     "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"):
            for i, n in enumerate(names):
                if n == want:
                    out[want] = f"{vals[i]} {units[i]}".strip()
        # tensor-pipe activity (tcgen05 issue / UTC pipes), whatever names this ncu exposes
        for i, n in enumerate(names):
            if ("pipe_tensor" in n or "pipe_tc" in n or "pipe_uma" in n or "pipe_utc" in n) and (
                    n.endswith(".pct_of_peak_sustained_active") or n.endswith(".sum")):
                out[n] = f"{vals[i]} {units[i]}".strip()
    for k, v in out.items():
        print(f"{k:70s} {v}")
    sass = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = sass[1]
    ix = {n: i for i, n in enumerate(h)}
    data = [r for r in sass[2:] if len(r) == len(h)]
    S = lambda r: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)  # noqa: E731
    N = lambda r: int(r[ix["Instructions Executed"]] or 0)  # noqa: E731
    tot_s = sum(S(r) for r in data) or 1
    tot_n = sum(N(r) for r in data) or 1
    print(f"\ninstructions {tot_n/1e6:.1f}M, stall samples {tot_s}")
    print("top stall sites:")
    for r in sorted(data, key=S, reverse=True)[:15]:
        print(f"  {r[ix['Address']][-5:]} {100*S(r)/tot_s:5.1f}%  {r[ix['Source']][:70]}")
    ops = {}
    for r in data:
        op = r[ix["Source"]].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        o = o.split(".")[0]
        ops[o] = ops.get(o, 0) + N(r)
    print("instruction mix:")
    for o, n in sorted(ops.items(), key=lambda x: -x[1])[:14]:
        print(f"  {o:10s} {100*n/tot_n:5.1f}%")
    if "--json" in sys.argv:
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tb = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if key in out:
                v, u = out[key].split()
                tb += float(v.replace(",", "")) * mult.get(u, 1)
        out["dram_bytes_per_launch"] = tb
        out["report"] = rep
        json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
