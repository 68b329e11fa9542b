"""Summarise an ncu --set full report into profiles/ (run here, no GPU needed).

  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_full_summary.json \
         [--traffic profiles/ncu_traffic_sift_np16.json]

Per kernel (first captured launch of each name): duration, DRAM bytes read +
written (the roofline "traffic"), DRAM / L2 throughput, L2 hit rate, achieved
occupancy, registers, executed instructions and tensor-pipe utilisation.
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "instructions",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active": "tensor_inst_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "pipe_fp64_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1_lsu_wavefronts_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    traffic_out = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
        if name in res:
            continue
        k = {}
        for m, key in WANT.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if key in ("dram_read", "dram_write", "l2_bytes"):
                v *= SCALE.get(u, 1)
            if key == "duration":
                v *= SCALE.get(u, 1)
                key = "duration_ms"
            k[key] = v
        if "dram_read" in k and "dram_write" in k:
            k["dram_bytes_per_launch"] = k["dram_read"] + k["dram_write"]
        res[name] = k
    with open(out, "w") as f:
        json.dump({"report": rep, "note": "ncu --set full --clock-control none; per-launch values, cold cache "
                   "(ncu flushes caches between replays)", "kernels": res}, f, indent=1)
    if traffic_out:
        with open(traffic_out, "w") as f:
            keep = ("dram_bytes_per_launch", "l2_hit_pct", "issue_active_pct", "pipe_xu_pct", "pipe_fp64_pct",
                    "l1_lsu_wavefronts_pct", "achieved_occupancy_pct", "instructions")
            json.dump({"source": out, "kernels": {n: {k: v.get(k) for k in keep if v.get(k) is not None}
                                                  for n, v in res.items()}}, f, indent=1)
    for n, v in res.items():
        print("%-22s %8.1f us  dram %8.1f MB  dram%% %5.1f  L2hit %5.1f  tensor %s" % (
            n, v.get("duration_ms", 0) * 1e3, v.get("dram_bytes_per_launch", 0) / 1e6,
            v.get("dram_pct_of_peak", 0), v.get("l2_hit_pct", 0), v.get("tensor_pipe_pct")))


if __name__ == "__main__":
    main()
