"""Summarise ncu captures (run here, on the CPU box) into profiles/*.json.

    python tools/ncu_summary.py <report.ncu-rep> <out.json> [launches.csv]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "smsp__average_warp_latency_issue_stalled_barrier": "stall_barrier",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "smsp__inst_executed.sum": "warp_instructions_executed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum": "smem_load_wavefronts",
    "sass__inst_executed_shared_loads": "smem_load_instructions",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_load_bank_conflicts",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_scoreboard",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier_per_issue",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio": "stall_no_instruction",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "stall_mio_throttle",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio": "stall_not_selected",
}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    unit = dict(zip(hdr, units))
    scale = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        m = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in KEYS.items():
            if k in d:
                try:
                    m[name] = float(d[k].replace(",", "")) * scale.get(unit.get(k, ""), 1)
                except ValueError:
                    m[name] = d[k]
        res.append(m)
    return res


def launch_list(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = None
    out = {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        e = out.setdefault(k, {"launches": 0, "total_ns": 0.0})
        e["launches"] += 1
        e["total_ns"] += v
    tot = sum(e["total_ns"] for e in out.values()) or 1.0
    for e in out.values():
        e["share"] = e["total_ns"] / tot
    return out


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    res = {"report": rep, "kernels": raw_metrics(rep)}
    for k in res["kernels"]:
        if "dram_read_bytes" in k and "dram_write_bytes" in k:
            k["dram_bytes_per_launch"] = k["dram_read_bytes"] + k["dram_write_bytes"]
    if len(sys.argv) > 3:
        res["launch_list"] = launch_list(sys.argv[3])
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
