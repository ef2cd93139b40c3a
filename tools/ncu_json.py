#!/usr/bin/env python3
"""Extract the roofline metrics of one kernel from an ncu --set full report into
the JSON committed under profiles/ (read by bench.py's roofline.traffic).
Usage: ncu_json.py report.ncu-rep kernel_regex out.json "command"
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_bytes.sum", "launch__block_size",
        "launch__grid_size", "launch__registers_per_thread",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed")

rep, rx, out, cmd = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{rx}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {}
for h, u, v in zip(hdr, units, vals):
    if any(h.endswith(k) for k in KEYS):
        d[h] = {"value": v, "unit": u}
d["_command"] = cmd
d["_note"] = "one launch, ncu --set full --clock-control none; values as reported by ncu -i --page raw"
json.dump(d, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in d.items() if not k.startswith("_")}, indent=0)[:1500])
