"""DRAM bytes per launch of the bench's kernels from an `ncu --set full`
capture -> profiles/ncu_traffic.json (bench.py fills roofline.traffic).

    python tools/ncu_traffic.py gpurun_out/full.ncu-rep [profiles/ncu_traffic.json]
"""
import csv
import io
import json
import re
import subprocess
import sys

NAMES = {"k_assemble_edges": "assemble_edges", "k_objective_seg": "objective",
         "k_objective": "objective", "k_corr_mma": "corr", "k_corr": "corr",
         "k_key_blocks": "key_blocks", "k_spd_factor": "spd_factor",
         "k_incidences": "incidences", "k_coords_sel": "coords",
         "k_assemble_edges_loc": "assemble_edges", "k_corr_tma": "corr", "k_rows": "rows",
         "k_var_rhs": "var_rhs", "k_spd_schur": "spd_schur", "k_incidences2": "incidences",
         "k_assemble_edges_stg": "assemble_edges"}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, out="profiles/ncu_traffic.json"):
    text = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                          text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    ri, wi = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    res = {}
    for r in rows[2:]:
        m = re.search(r"(k_\w+)", r[ki])
        if not m or m.group(1) not in NAMES:
            continue
        b = (float(r[ri].replace(",", "")) * SCALE.get(units[ri], 1.0)
             + float(r[wi].replace(",", "")) * SCALE.get(units[wi], 1.0))
        res.setdefault(NAMES[m.group(1)], []).append(b)
    summary = {k: max(v) for k, v in res.items()}   # level-1 launch for spd_factor
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
