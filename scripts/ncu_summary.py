"""Summarise an ncu --set full report (per kernel: time, DRAM bytes, tensor/L2/DRAM
utilisation, registers) as markdown; also emits a JSON of per-kernel DRAM traffic."""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = {
    "time_us": r"^gpu__time_duration.sum$",
    "dram_read_MB": r"^dram__bytes_read.sum$",
    "dram_write_MB": r"^dram__bytes_write.sum$",
    "tensor_pct": r"^sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed$",
    "l2_pct": r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$",
    "dram_pct": r"^gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed$",
    "sm_clock_GHz": r"^sm__cycles_elapsed.avg.per_second$",
    "regs": r"^launch__registers_per_thread$",
    "grid": r"^launch__grid_size$",
}
SCALE = {"us": 1.0, "ms": 1e3, "ns": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Kbyte": 1e-3, "byte": 1e-6,
         "Ghz": 1.0, "Mhz": 1e-3, "%": 1.0}


def main(rep, out_md, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    cols = {k: next((i for i, x in enumerate(h) if re.search(p, x)), None) for k, p in KEYS.items()}
    ki = h.index("Kernel Name")
    lines = ["| kernel | time us | DRAM read MB | DRAM write MB | tensor % | L2 % | DRAM % | SM GHz | regs | grid |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = []
    for r in data:
        vals = {}
        for k, i in cols.items():
            if i is None or not r[i]:
                vals[k] = None
                continue
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                vals[k] = r[i]
                continue
            vals[k] = v * SCALE.get(units[i], 1.0)
        name = re.sub(r"\(CUtensorMap_st.*|\(.*", "", r[ki])[:70]
        fmt = lambda v, p=1: "-" if v is None else (f"{v:.{p}f}" if isinstance(v, float) else str(v))  # noqa: E731
        lines.append(f"| `{name}` | {fmt(vals['time_us'])} | {fmt(vals['dram_read_MB'])} | {fmt(vals['dram_write_MB'])} | "
                     f"{fmt(vals['tensor_pct'])} | {fmt(vals['l2_pct'])} | {fmt(vals['dram_pct'])} | "
                     f"{fmt(vals['sm_clock_GHz'], 2)} | {fmt(vals['regs'], 0)} | {fmt(vals['grid'], 0)} |")
        traffic.append({"kernel": name, "time_us": vals["time_us"],
                        "dram_bytes": (vals["dram_read_MB"] or 0) * 1e6 + (vals["dram_write_MB"] or 0) * 1e6})
    open(out_md, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(out_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
