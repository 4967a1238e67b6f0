"""Generate golden fixtures from the REAL reference package.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    python oracle/make_golden.py

It imports the reference package under the name ``mosaic_ref`` (so it can
never shadow anything in this repo), runs its own hot-path operator and
schedule code on seeded inputs, and writes the inputs and outputs as small
fixtures under tests/golden/. The tests then pin both the CPU oracle and the
CUDA path against these files.
"""
from __future__ import annotations

import importlib.util
import json
import random
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src/mosaic")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "mosaic_ref", REF_SRC / "__init__.py", submodule_search_locations=[str(REF_SRC)]
    )
    mod = importlib.util.module_from_spec(spec)
    sys.modules["mosaic_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def kernel_cases(ref) -> dict[str, np.ndarray]:
    """Seeded gather_gemm problems in the style of tests/test_kernel.py:38-53."""
    from mosaic_ref.kernel import GatherGemmProblem, gather_gemm

    arrays: dict[str, np.ndarray] = {}
    rng = random.Random(2601)
    for case in range(40):
        n = rng.randint(1, 12)
        d = rng.randint(1, 9)
        V = rng.randint(1, 15)
        hidden = np.array([[rng.uniform(-3, 3) for _ in range(d)] for _ in range(n)])
        weight = np.array([[rng.uniform(-3, 3) for _ in range(V)] for _ in range(d)])
        m = rng.randint(1, n)
        idx = np.array(rng.sample(range(n), m), dtype=np.int64)
        tiles = np.array([rng.randint(1, 5), rng.randint(1, 5), rng.randint(1, 5)], dtype=np.int64)
        out, scratch = gather_gemm(GatherGemmProblem(hidden, weight, tuple(int(i) for i in idx), *map(int, tiles)))
        p = f"rand{case:02d}_"
        arrays[p + "hidden"] = hidden
        arrays[p + "weight"] = weight
        arrays[p + "idx"] = idx
        arrays[p + "tiles"] = tiles
        arrays[p + "out"] = out
        arrays[p + "scratch"] = np.array([scratch.peak_elements, scratch.bound], dtype=np.int64)
    # a bf16-representable medium case the GPU path can also be pinned on:
    g = np.random.default_rng(2602)
    from mosaic_oracle import bf16_round  # noqa: E402  (oracle is on sys.path)

    hidden = bf16_round(g.standard_normal((96, 128)))
    weight = bf16_round(g.standard_normal((128, 520)) * 0.05)
    idx = g.choice(96, size=40, replace=False).astype(np.int64)
    out, _ = gather_gemm(GatherGemmProblem(hidden, weight, tuple(int(i) for i in idx), 32, 32, 32))
    arrays["bf16case_hidden"] = hidden
    arrays["bf16case_weight"] = weight
    arrays["bf16case_idx"] = idx
    arrays["bf16case_out"] = out
    return arrays


def schedule_cases(ref) -> list[dict]:
    from mosaic_ref.workload import ScenarioConfig

    cases = []
    for L, rp, N in [(10, 0.2, 4), (2048, 0.5, 64), (32768, 0.5, 64), (65536, 0.5, 48),
                     (131072, 0.5, 128), (1000, 0.37, 7), (7, 0.0, 3), (4096, 0.25, 100)]:
        sc = ScenarioConfig(length=L, prompt_ratio=rp, steps=N)
        cases.append({
            "L": L, "prompt_ratio": rp, "steps": N,
            "output_length": sc.output_length,
            "masked_at": [sc.masked_at(n) for n in range(N + 1)],
        })
    return cases


def main() -> None:
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    ref = load_reference()
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "kernel_golden.npz", **kernel_cases(ref))
    with open(OUT / "sched_golden.json", "w") as f:
        json.dump(schedule_cases(ref), f, indent=1)
        f.write("\n")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
