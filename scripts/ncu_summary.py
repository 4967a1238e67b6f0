"""Summarise an ncu --set full capture of one kernel into a small JSON (kept
under profiles/): duration, clocks, DRAM traffic per launch, L2 and tensor-pipe
figures. Usage: python scripts/ncu_summary.py REP.ncu-rep OUT.json [--traffic]
(--traffic also writes profiles/k3_traffic.json, read by bench.py)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = {
    "kernel": "Kernel Name",
    "duration_ns": "gpu__time_duration.sum",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_bytes": "lts__t_bytes.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l2_fabric_sectors": "lts__t_sectors_srcunit_ltcfabric.sum",
    "tensor_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_dynamic": "launch__shared_mem_per_block_dynamic",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e6, "us": 1e3, "ns": 1,
         "Ghz": 1e9, "Mhz": 1e6, "hz": 1, "Tbyte": 1e12}


def main():
    rep, out = sys.argv[1], Path(sys.argv[2])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {}
        for k, name in KEYS.items():
            if name not in hdr:
                continue
            i = hdr.index(name)
            v = vals[i]
            try:
                f = float(v.replace(",", ""))
                f *= SCALE.get(units[i], 1)
                d[k] = f
            except ValueError:
                d[k] = v
        launches.append(d)
    summary = {"source": rep, "launches": launches}
    out.write_text(json.dumps(summary, indent=1))
    if "--traffic" in sys.argv:
        sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
        from paper_2601_06562_b200 import _build

        l0 = launches[0]
        t = {"bytes_per_launch": l0["dram_read_bytes"] + l0["dram_write_bytes"],
             "kernel": l0.get("kernel"), "source": f"profiles/{out.name}", "duration_ns_under_ncu": l0.get("duration_ns"),
             "code_hash": _build.source_hash(_build.K3_SOURCES),
             "code_hash_of": "csrc/lmhead.cu + csrc/common.cuh + nvcc flags (paper_2601_06562_b200._build.source_hash)"}
        (out.parent / "k3_traffic.json").write_text(json.dumps(t, indent=1))
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
