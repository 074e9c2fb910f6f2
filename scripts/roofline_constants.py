"""Derive bench.py's roofline constants from a committed ncu metrics capture of ONE full-size E-step
launch, and write them to profiles/roofline_constants.json (bench.py reads that file; nothing is
typed in by hand, so the fraction recomputes from the capture).

    python scripts/roofline_constants.py NAME CAPTURE.csv PAIRS [--note TEXT]

CAPTURE.csv: `ncu --csv --metrics <METRICS> -k regex:estep_ -c 1 ...` output (one kernel), e.g.
profiles/r02_ncu_metrics_cfg5.csv, or an .ncu-rep (--set full).  PAIRS = n * g of that launch.
--bytes-scale: the capture covered a slice of the bench launch (n_full / n_slice for the DRAM bytes;
the flops are per pair).
  flops_per_pair  = (2 dfma + dadd + dmul) / PAIRS      (executed FP64 flops, thread level)
  dram bytes      = dram__bytes_read.sum + dram__bytes_write.sum of the launch
  fp64_pipe_active= sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active / 100
"""
import argparse
import csv
import io
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "roofline_constants.json")
METRICS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
           "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
           "sm__warps_active.avg.per_cycle_active"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0, "inst": 1.0, "%": 1.0, "": 1.0}


def parse_rep(path):
    """An ncu report (--set full) or its exported raw page (`ncu -i REP --page raw --csv`, one kernel)
    -> {metric: value in base units}."""
    if path.endswith(".ncu-rep"):
        import subprocess
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    else:
        out = open(path).read()
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            d[h] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
        except ValueError:
            pass
    # --set full stores the sass counters as per-cycle rates: x cycles elapsed
    cyc = d.get("sm__cycles_elapsed.avg")
    for op in ("dfma", "dadd", "dmul"):
        k = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum"
        if k not in d and k + ".per_cycle_elapsed" in d:
            d[k] = d[k + ".per_cycle_elapsed"] * cyc
    return vals[hdr.index("Kernel Name")], d


def parse(path):
    """ncu --csv (metrics, one row per metric) -> {metric: value in base units}; or an .ncu-rep."""
    text = open(path).read()
    hdr_line = next((l for l in text.split("\n") if l.startswith('"ID"')), "")   # ncu's banner lines may precede it
    if path.endswith(".ncu-rep") or '"Metric Name"' not in hdr_line:
        return parse_rep(path)
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    out, kernel = {}, None
    for r in rows:
        kernel = kernel or r.get("Kernel Name")
        v = r["Metric Value"].replace(",", "")
        try:
            out[r["Metric Name"]] = float(v) * SCALE.get(r.get("Metric Unit", ""), 1.0)
        except ValueError:
            pass
    return kernel, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("capture")
    ap.add_argument("pairs", type=float)
    ap.add_argument("--note", default="")
    ap.add_argument("--bytes-scale", type=float, default=1.0,
                    help="scale the DRAM bytes (capture on a slice of the launch: n_full / n_slice)")
    a = ap.parse_args()
    kernel, m = parse(a.capture)
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m[k] *= a.bytes_scale
    flops = (2 * m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
             + m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
             + m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"])
    entry = {"kernel": kernel, "source": os.path.relpath(a.capture, ROOT), "pairs": a.pairs,
             "flops_per_pair": flops / a.pairs, "fp64_flops": flops,
             "dram_read_bytes": m["dram__bytes_read.sum"], "dram_write_bytes": m["dram__bytes_write.sum"],
             "dram_bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
             "fp64_pipe_active": m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0) / 100.0,
             "ncu_duration_s": m.get("gpu__time_duration.sum"),
             "ncu_flop_rate_tflops": flops / m["gpu__time_duration.sum"] / 1e12 if m.get("gpu__time_duration.sum") else None,
             "registers": m.get("launch__registers_per_thread"), "warps_active": m.get("sm__warps_active.avg.per_cycle_active"),
             "bytes_scale": a.bytes_scale, "note": a.note}
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    data[a.name] = entry
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
