"""Fold ncu captures of the fp32 kernel into the committed summaries:
  python tools/fold_fp32_captures.py <rank_plans_f32.csv> <fp32_full_raw.csv>
* rank_plans csv: `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
  gpu__time_duration.sum --csv` of `tools/rank_plan_once.py f32 32768 1 2 4 8`
  -> the fp32 rows of profiles/r02_ncu_summary.json (bench.py's roofline.traffic);
* fp32_full_raw csv: `ncu -i <rep> --page raw --csv` of the `--set full` capture
  of tools/headline_once.py's second sgemm launch -> profiles/r02_ncu_full_summary.json."""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PLAN = "sgemm_tma_kernel<128x256, FFMA2, A k-major>"
N = 32768


def rank_plans(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    launch = {}
    for r in csv.DictReader(io.StringIO("".join(lines))):
        d = launch.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    seq = [launch[i] for i in sorted(launch)]
    gem = [x for x in seq if "sgemm_tma_kernel" in x["name"]]
    tr = [x for x in seq if "transpose_f32" in x["name"]]
    p = os.path.join(ROOT, "profiles", "r02_ncu_summary.json")
    S = json.load(open(p))
    S["kernels"] = [k for k in S["kernels"] if k.get("dtype") != "f32"]
    gi = 0
    for P_, cnt in ((1, 1), (2, 2), (4, 2), (8, 2)):
        g, t = gem[gi:gi + cnt], tr[gi:gi + cnt]
        gi += cnt
        rows0 = N // P_
        rd = sum(x["dram__bytes_read.sum"] for x in g)
        wr = sum(x["dram__bytes_write.sum"] for x in g)
        ns = sum(x["gpu__time_duration.sum"] for x in g)
        tns = sum(x["gpu__time_duration.sum"] for x in t)
        alg = 4 * (2 * rows0 * N + N * N)
        S["kernels"].append({
            "n": N, "rows": rows0, "P": P_, "dtype": "f32", "role": "dominant", "plan": PLAN,
            "launches": cnt, "dram_bytes": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "ncu_ms": ns / 1e6, "algorithmic_bytes": alg, "traffic_over_algorithmic": (rd + wr) / alg,
            "ncu_tflops": 2.0 * rows0 * N * N / (ns / 1e9) / 1e12,
            "transpose_pass": {
                "launches": len(t), "ncu_ms": tns / 1e6,
                "dram_bytes": sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in t),
                "share_of_multiply_time": tns / ns}})
    json.dump(S, open(p, "w"), indent=1)
    for k in S["kernels"][-4:]:
        print(k["P"], round(k["ncu_tflops"], 2), "TFLOP/s", round(k["dram_bytes"] / 1e9, 1), "GB",
              "transpose %.2f%%" % (100 * k["transpose_pass"]["share_of_multiply_time"]))


def full(path):
    rows = list(csv.reader(open(path)))
    hdr, vals = rows[0], rows[2]
    p = os.path.join(ROOT, "profiles", "r02_ncu_full_summary.json")
    S = json.load(open(p))
    old = [k for k in S["kernels"] if "row_major" in k["capture"] or k["capture"] == "r02_fp32"][0]
    if old["capture"] == "r02_fp32":
        old["capture"] = ("r02_fp32_row_major (the earlier instance, A staged as it lies, 4-stage "
                          "ring; kept for comparison)")
    S["kernels"] = [k for k in S["kernels"] if "k-major" not in k["capture"]]
    new = {"kernel": vals[hdr.index("Kernel Name")][:90],
           "capture": "r02_fp32 (A k-major instance, 3-stage ring, N=16384)"}
    keys = [k for k in old if k not in ("kernel", "capture")] + [
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"]
    for key in keys:
        if key in hdr:
            new[key] = float(vals[hdr.index(key)].replace(",", ""))
    S["kernels"].append(new)
    json.dump(S, open(p, "w"), indent=1)
    print({k: new[k] for k in new if "fma" in k or "issue_active" in k or "duration" in k})


if __name__ == "__main__":
    rank_plans(sys.argv[1])
    full(sys.argv[2])
