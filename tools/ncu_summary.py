"""Summarise one `ncu --set full` capture of the frames kernel into profiles/<out>.json.
usage: python tools/ncu_summary.py gpurun_out/X_frames.ncu-rep profiles/X_frames_ncu.json "label" """
import csv
import json
import subprocess
import sys

rep, out, label = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]


def g(n):
    return v[h.index(n)]


dur = float(g("gpu__time_duration.sum"))
dur_ms = dur / 1e3 if u[h.index("gpu__time_duration.sum")] == "us" else dur
rd, wr = float(g("dram__bytes_read.sum")), float(g("dram__bytes_write.sum"))
scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}
rd_b = rd * scale[u[h.index("dram__bytes_read.sum")]]
wr_b = wr * scale[u[h.index("dram__bytes_write.sum")]]
res = {
    "kernel": label,
    "command": "ncu --set full --import-source on --clock-control none -k regex:frames_small -c 1 "
               "python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity",
    "gpu__time_duration_ms": dur_ms,
    "dram__bytes_read_MB": rd_b / 1e6,
    "dram__bytes_write_MB": wr_b / 1e6,
    "traffic_bytes_per_launch": int(rd_b + wr_b),
    "sm__warps_active_pct": float(g("sm__warps_active.avg.pct_of_peak_sustained_active")),
    "smsp__issue_active_pct": float(g("smsp__issue_active.avg.pct_of_peak_sustained_active")),
    "lts__t_sector_hit_rate_pct": float(g("lts__t_sector_hit_rate.pct")),
    "l1tex__t_sector_hit_rate_pct": float(g("l1tex__t_sector_hit_rate.pct")),
    "registers_per_thread": int(float(g("launch__registers_per_thread"))),
    "inst_executed": int(float(g("smsp__inst_executed.sum"))),
    "grid": g("launch__grid_size"), "block": g("launch__block_size"),
    "shared_mem_per_block_dynamic_KB": g("launch__shared_mem_per_block_dynamic"),
}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
