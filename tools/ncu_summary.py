"""Summarise an `ncu --set full` report (ncu -i <rep> --page raw --csv) into the
JSON kept under profiles/: per kernel launch its duration, DRAM bytes, the
fraction of peak for its roofline, and the main utilisation/stall metrics.

    python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep profiles/ncu_r01_full.json \
        [--leaf-json profiles/ncu_leaf.json]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1.0),
    "dram_read_gb": ("dram__bytes_read.sum", 1.0),
    "dram_write_gb": ("dram__bytes_write.sum", 1.0),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dmma_pipe_pct_active": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1.0),
    "stall_math_throttle": ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", 1.0),
    "stall_wait": ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", 1.0),
    "stall_short_scoreboard": ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", 1.0),
    "stall_long_scoreboard": ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", 1.0),
}
UNIT_SCALE = {"ms": 1.0, "msecond": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6,
              "s": 1e3, "second": 1e3, "Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9,
              "Tbyte": 1e3}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--leaf-json")
    ap.add_argument("--hbm-gbs", type=float, default=6547.2)
    a = ap.parse_args()
    hdr, units, data = load(a.rep)
    idx = {h: i for i, h in enumerate(hdr)}
    launches = []
    for d in data:
        rec = {"kernel": d[idx["Kernel Name"]].split("(")[0].strip()}
        for k, (metric, _) in KEYS.items():
            if metric not in idx:
                continue
            v = d[idx[metric]].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[idx[metric]]
            if k.endswith("_ms") or k.endswith("_gb"):
                x *= UNIT_SCALE.get(u, 1.0)
            rec[k] = x
        if "dram_read_gb" in rec and "duration_ms" in rec:
            rec["dram_gbs"] = (rec["dram_read_gb"] + rec["dram_write_gb"]) / (rec["duration_ms"] * 1e-3)
            rec["dram_frac_of_measured_hbm"] = rec["dram_gbs"] / a.hbm_gbs
        launches.append(rec)
    json.dump({"report": a.rep, "launches": launches}, open(a.out, "w"), indent=1)
    if a.leaf_json:
        leaf = [l for l in launches if "leaf" in l["kernel"]]
        if leaf:
            l0 = leaf[0]
            json.dump({"kernel": l0["kernel"], "dram_bytes_per_launch":
                       (l0["dram_read_gb"] + l0["dram_write_gb"]) * 1e9,
                       "dram_read_bytes": l0["dram_read_gb"] * 1e9,
                       "dram_write_bytes": l0["dram_write_gb"] * 1e9,
                       "duration_ms_ncu": l0["duration_ms"], "source": a.out},
                      open(a.leaf_json, "w"), indent=1)
    for l in launches:
        print(json.dumps(l))


if __name__ == "__main__":
    main()
