"""Summarise an ncu report (`ncu -i X.ncu-rep --page raw --csv`) into JSON: per launch the
duration, DRAM bytes, SM / DRAM throughput, tensor (DMMA / int8) and fp64 pipe activity,
occupancy, registers and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/r02/latency_cfg4.ncu-rep "about text" > profiles/x.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dram_throughput_pct": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "grid_size": ("launch__grid_size", 1.0),
    "block_size": ("launch__block_size", 1.0),
    "sm_clock_ghz": ("smsp__cycles_elapsed.avg.per_second", 1.0),
}
STALL, STALL_END = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
# unit -> factor to the key's unit (us, bytes, GHz)
UNIT = {"nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "ns": 1e-3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main():
    rep, about = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = {"_about": about, "_source": rep}
    for i, row in enumerate(data):
        name = row[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        d = {}
        for k, (m, sc) in KEYS.items():
            if m in hdr:
                v = num(row[hdr.index(m)])
                if v is not None:
                    d[k] = round(v * sc * UNIT.get(units[hdr.index(m)], 1.0), 4)
        if "dram_read_bytes" in d and "dram_write_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        stalls = []
        for j, k in enumerate(hdr):
            if k.startswith(STALL) and k.endswith(STALL_END) and "selected" not in k:
                v = num(row[j])
                if v:
                    stalls.append((v, k[len(STALL):-len(STALL_END)]))
        d["top_stalls_cycles_per_issue"] = {k: round(v, 2) for v, k in sorted(stalls, reverse=True)[:5]}
        out[f"launch {i}: {name}"] = d
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
