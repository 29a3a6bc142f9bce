"""Summarise an `ncu --set full` capture (.ncu-rep) per kernel launch.

    python tools/ncu_summary.py gpurun_out/full_r01.ncu-rep [out.txt]

Prints, per captured launch: duration, DRAM bytes (read + write = the
`roofline.traffic` figure), achieved DRAM GB/s, FP64 pipe / FP64 tensor
utilisation, occupancy, registers, and the L1/L2 hit rates.
"""
import csv
import io
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe%"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "dmma%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
]
SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "s": 1.0, "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name):
    m = re.search(r"(k_\w+(<[^>]*>)?|Device\w+Kernel|\w+_kernel)", name)
    return m.group(1) if m else name[:40]


def main(path, out=None):
    text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                          text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    lines = [f"# {path}: per-launch summary (ncu --set full, --clock-control none)",
             f"{'kernel':34s} {'dur_us':>9s} {'dram_MB':>9s} {'GB/s':>8s} " +
             " ".join(f"{lab:>9s}" for _, lab in METRICS[3:])]
    for r in rows[2:]:
        vals = {}
        for name, lab in METRICS:
            if name not in h:
                vals[lab] = None
                continue
            i = h.index(name)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                vals[lab] = None
                continue
            vals[lab] = v * SCALE.get(units[i], 1.0) if lab in ("dur", "dram_rd", "dram_wr") else v
        dur = vals["dur"] or float("nan")
        traffic = (vals["dram_rd"] or 0.0) + (vals["dram_wr"] or 0.0)
        rest = " ".join(f"{(vals[lab] if vals[lab] is not None else float('nan')):9.1f}"
                        for _, lab in METRICS[3:])
        lines.append(f"{short(r[ki]):34s} {dur * 1e6:9.1f} {traffic / 1e6:9.1f} "
                     f"{traffic / dur / 1e9:8.0f} {rest}")
    txt = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(txt)
    print(txt, end="")


if __name__ == "__main__":
    main(*sys.argv[1:])
