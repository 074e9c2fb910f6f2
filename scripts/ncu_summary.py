"""Summarise an ncu --set full report of the E-step kernel into a committed text file:
key throughput metrics, executed FP64 flops (2*dfma + dadd + dmul), stall reasons, opcode mix."""
import collections
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, pairs, out):
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    d = dict(zip(hdr, vals))
    unit = dict(zip(hdr, units))
    cyc = float(d["sm__cycles_elapsed.avg"])
    f = lambda k: float(d[k]) * cyc
    fma = f("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed")
    add = f("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed")
    mul = f("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed")
    flops = 2 * fma + add + mul
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}
    dur = float(d["gpu__time_duration.sum"]) * scale.get(unit.get("gpu__time_duration.sum", "ms"), 1e-3)
    lines = [f"report: {rep}", f"kernel: {vals[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else '?'}",
             f"duration_ms: {dur * 1e3:.4f}   sm_cycles: {cyc:.0f}",
             f"fp64 executed flops (2*dfma+dadd+dmul): {flops:.4e}   per pair ({pairs} pairs): {flops / pairs:.4e}",
             f"fp64 achieved: {flops / dur / 1e12:.2f} TFLOP/s   flop fraction of 148x64x2/clk: {flops / cyc / 18944:.3f}"]
    for k in ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed.sum.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
              "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.per_cycle_active",
              "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"]:
        lines.append(f"{k}: {d.get(k)} {unit.get(k, '')}")
    lines.append("stall reasons (warps per issue-active cycle):")
    for h, v in zip(hdr, vals):
        if "average_warps_issue_stalled" in h and h.endswith("ratio"):
            try:
                if float(v) > 0.02:
                    lines.append(f"  {h.split('stalled_')[1].split('_per')[0]}: {float(v):.3f}")
            except ValueError:
                pass
    sass = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    sh = sass[1]
    rows = [dict(zip(sh, r)) for r in sass[2:] if len(r) == len(sh)]
    tot = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    ins = sum(float(r["Instructions Executed"] or 0) for r in rows)
    by_s, by_i = collections.Counter(), collections.Counter()
    for r in rows:
        toks = r["Source"].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
        by_s[op] += float(r["Warp Stall Sampling (All Samples)"] or 0)
        by_i[op] += float(r["Instructions Executed"] or 0)
    lines.append("opcode mix (share of warp-stall samples / of executed warp instructions):")
    for op, v in by_s.most_common(20):
        lines.append(f"  {op:10s} {100 * v / tot:5.1f}%  {100 * by_i[op] / ins:5.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:6]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
