"""Summarise an ncu report (.ncu-rep) into profiles/: per-kernel key metrics,
stall breakdown and DRAM traffic per launch.  Runs here (no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_c4 [--config c4]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "sm__inst_executed.avg.per_cycle_active": "ipc_per_sm",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_inst_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_cycles_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return f * scale


def main():
    rep, out = sys.argv[1], sys.argv[2]
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else None
    kernels = []
    for d, u in raw(rep):
        k = {"kernel": d.get("Kernel Name", "")[:120]}
        for m, name in KEYS.items():
            if m in d and d[m] not in ("", "n/a"):
                if name.startswith("dram"):
                    k[name + "_bytes"] = to_bytes(d[m], u.get(m, "byte"))
                elif name == "duration":
                    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "s": 1e6}.get(u.get(m), 1)
                    k["duration_us"] = float(d[m].replace(",", "")) * scale
                else:
                    try:
                        k[name] = float(d[m].replace(",", ""))
                    except ValueError:
                        k[name] = d[m]
        stalls = {}
        for m, v in d.items():
            if m.startswith("smsp__average_warps_issue_stalled") and m.endswith("_per_issue_active.ratio"):
                try:
                    val = float(v)
                except ValueError:
                    continue
                if val > 0.02:
                    stalls[m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(val, 3)
        k["stalls_per_issue"] = stalls
        if "dram_read_bytes" in k:
            k["traffic_bytes"] = k["dram_read_bytes"] + k.get("dram_write_bytes", 0.0)
        kernels.append(k)
    with open(out + ".json", "w") as f:
        json.dump({"report": rep, "kernels": kernels}, f, indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu summary: {rep}\n\n")
        f.write("| kernel | us | regs | warps/SM | IPC | issue% | XU% | FMA cyc% | DRAM B (r+w) |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for k in kernels:
            f.write(f"| {k['kernel'][:60]} | {k.get('duration_us', 0):.1f} | {k.get('registers', '')} | "
                    f"{k.get('warps_active_per_sm', 0):.2f} | {k.get('ipc_per_sm', 0):.2f} | "
                    f"{k.get('issue_active_pct', 0):.1f} | {k.get('xu_pipe_pct', 0):.1f} | "
                    f"{k.get('fma_pipe_cycles_pct', 0):.1f} | {k.get('traffic_bytes', 0):.3g} |\n")
        f.write("\nStalls (cycles per issued instruction):\n\n")
        for k in kernels:
            f.write(f"- {k['kernel'][:60]}: {k['stalls_per_issue']}\n")
    if cfg:  # traffic per launch of the dominant (longest) kernel, read by bench.py
        dom = max(kernels, key=lambda k: k.get("duration_us", 0))
        path = "profiles/ncu_traffic.json"
        try:
            cur = json.load(open(path))
        except (OSError, ValueError):
            cur = {}
        cur[cfg] = dom.get("traffic_bytes")
        json.dump(cur, open(path, "w"), indent=1)
    print(open(out + ".md").read())


if __name__ == "__main__":
    main()
