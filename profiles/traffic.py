"""Per-stage DRAM traffic from an ncu ``--set full`` report.

Usage: python profiles/traffic.py <report.ncu-rep> <workload> <precision>
Merges {"<workload>/<precision>": {stage: bytes_per_launch}} into
profiles/dram_traffic.json (read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys

STAGE = {
    "k_spread_tiles": "spread", "k_spread_warp": "spread", "k_combine": "combine", "k_x_comb_r2c": "fft_x", "k_x_bulk_r2c": "fft_x", "k_x_r2c": "fft_x",
    "k_y_fwd": "fft_y", "k_z_reduce": "fft_z_scale_reduce", "k_z_ik": "ifft_z_ik",
    "k_y_inv": "ifft_y", "k_x_c2r": "ifft_x", "k_xy_fwd": "fft_xy", "k_yx_inv": "ifft_yx", "k_gather_warp": "gather",
    "k_gather_ik": "gather", "k_gather_tma": "gather", "k_scale_reduce": "scale_reduce",
    "k_bin_keys": "bin_keys", "k_bin_gather": "bin_gather", "k_bin_records_u": "bin_records",
    "k_bin_sorted": "bin_gather_weights",
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, workload, precision):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    # per kernel instantiation: mean over its captured launches; a stage that
    # runs as several instantiations per step (the bulk-staged x pass: one
    # launch per z-plane class) is their sum
    acc = {}
    for r in data:
        full = r[ki].split("(")[0].replace("void ", "").strip()
        base = full.split("<")[0].split("::")[-1].strip()
        st = STAGE.get(base)
        if not st:
            continue
        b = (float(r[rd].replace(",", "")) * SCALE[units[rd]] +
             float(r[wr].replace(",", "")) * SCALE[units[wr]])
        acc.setdefault(st, {}).setdefault(full, []).append(b)
    res = {k: int(sum(sum(v) / len(v) for v in inst.values())) for k, inst in acc.items()}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dram_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[f"{workload}/{precision}"] = res
    with open(path, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*sys.argv[1:4])
