"""Extract per-kernel DRAM traffic from `ncu --set full` reports into
profiles/<round>_traffic.json (read by bench.py for roofline.traffic).

usage: python tools/ncu_traffic.py OUT.json REPORT.ncu-rep [...]
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def one(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]

    def get(name):
        if name not in h:
            return None
        i = h.index(name)
        return float(v[i].replace(",", "")) * SCALE.get(u[i], 1)

    name = v[h.index("Kernel Name")]
    base = name.split("(")[0].split("<")[0].replace("void ", "").replace("fs4d::", "").strip()
    pct = {k: get(m) for k, m in (
        ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("mem_throughput_pct", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"))}
    return base, {"kernel": name[:100], "dram_read_bytes": get("dram__bytes_read.sum"),
                  "dram_write_bytes": get("dram__bytes_write.sum"), "duration_s": get("gpu__time_duration.sum"),
                  "utilisation": pct, "source": path.split("/")[-1]}


def main():
    out = {}
    for p in sys.argv[2:]:
        k, d = one(p)
        out[k] = d
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
