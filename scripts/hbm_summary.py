"""HBM-bound kernels from an ncu --set full capture of scripts/ncu_targets.py
(summarised by scripts/ncu_summary.py): measured DRAM bytes and algorithmic
bytes per launch, GB/s against the measured copy bandwidth.

    python scripts/hbm_summary.py SUMMARY.json [MEASURED_PEAKS.json]
"""
import json
import re
import sys

# algorithmic bytes per launch at the shapes of scripts/ncu_targets.py
ALGO = {
    "k2_gather": 2 * 16384 * 4096 * 2,               # read + write 16384 rows of d 4096 bf16
    "k11_rope": 2 * 2 * 32768 * 4096 * 2,            # q and k read + written
    "k6_swiglu": 3 * 32768 * 12288 * 2,              # gate, up read; act written
    "k9_combine": (8 + 1) * 65536 * 2048 * 2 + 65536 * 8 * 8,  # top-8 rows read, one written; pos + weight
}
FLOPS = {"k10_ffn_gemm": [2 * 2 * 32768 * 4096 * 12288, 2 * 32768 * 12288 * 4096]}  # gate/up+SwiGLU, down+residual


def main():
    s = json.load(open(sys.argv[1]))
    peaks = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else {}
    hbm = peaks.get("hbm_gbs", 6552.6)
    seen = {}
    for l in s["launches"]:
        m = re.search(r"(k\d+_[a-z0-9_]+)", l["kernel"])
        name = m.group(1) if m else l["kernel"][:14]
        ns = l["duration_ns"]
        dram = l.get("dram_read_bytes", 0) + l.get("dram_write_bytes", 0)
        line = f"{name:14s} {ns / 1e3:9.1f} us  DRAM {dram / 1e9:6.3f} GB = {dram / ns:6.0f} GB/s ({dram / ns / hbm:.2f} of measured {hbm:.0f} GB/s)"
        key = next((k for k in ALGO if name.startswith(k)), None)
        if key:
            line += f"  algorithmic {ALGO[key] / 1e9:.3f} GB -> {ALGO[key] / ns:6.0f} GB/s ({ALGO[key] / ns / hbm:.2f})"
        if name.startswith("k10"):
            i = seen.get("k10", 0)
            seen["k10"] = i + 1
            f = FLOPS["k10_ffn_gemm"][min(i, 1)]
            line += f"  {f / ns / 1e3:.0f} TFLOP/s  tensor pipe {l.get('tensor_active_pct', 0):.1f}%"
        print(line + f"  SM {l.get('sm_clock_hz', 0) / 1e6:.0f} MHz  regs {l.get('registers', 0):.0f}")


if __name__ == "__main__":
    main()
