"""Summarise an ncu report (raw page) into the JSON committed under profiles/."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores", "launch__occupancy_limit_registers",
        "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static"]


def summarize(rep, name):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": vals[i], "unit": units[i]}
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}
        rb, wb = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if rb and wb:
            d["dram_bytes_per_launch"] = (float(rb["value"].replace(",", "")) * scale[rb["unit"]]
                                          + float(wb["value"].replace(",", "")) * scale[wb["unit"]])
        out.append(d)
    res = {"report": name, "launches": out,
           "dram_bytes_per_launch": out[0].get("dram_bytes_per_launch") if out else None}
    return res


if __name__ == "__main__":
    print(json.dumps(summarize(sys.argv[1], sys.argv[2]), indent=1))
