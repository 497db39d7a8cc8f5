"""Per-kernel key metrics of an ncu --set full capture (profiles/ evidence):
duration, DRAM bytes and bandwidth, L2 hit rate, occupancy, FP64 pipe and
FP64 tensor-core (DMMA) utilisation.

    python tools/ncu_full_summary.py gpurun_out/r02c_full_C4.ncu-rep > profiles/r02c_full_C4.txt
"""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3),
        ("dram__bytes_read.sum", "MB rd", 1e-6),
        ("dram__bytes_write.sum", "MB wr", 1e-6),
        ("lts__t_sector_hit_rate.pct", "L2 hit%", 1.0),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1.0),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM%", 1.0),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "fp64 pipe%", 1.0),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA%act", 1.0),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%el", 1.0)]
UNIT = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# {path}: {len(rows) - 2} kernel launches (ncu --set full, --clock-control none, serialised, cold L2)")
    print(f"{'kernel':34s} " + " ".join(f"{lab:>10s}" for _, lab, _ in COLS) + f" {'GB/s':>8s}")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("gn::<unnamed>::", "")
        vals = []
        for col, _, scale in COLS:
            i = idx.get(col)
            if i is None or not r[i]:
                vals.append(float("nan"))
                continue
            v = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
            vals.append(v * scale)
        gbs = (vals[1] + vals[2]) * 1e6 / (vals[0] * 1e-6) / 1e9 if vals[0] > 0 else float("nan")   # MB / us
        print(f"{name[:34]:34s} " + " ".join(f"{v:10.2f}" for v in vals) + f" {gbs:8.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
