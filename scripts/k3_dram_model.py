"""Wave model of K3's DRAM traffic under the die-aware unit schedule
(csrc/lmhead.cu unit_coords + the die split), for the DESIGN §4 analysis.

Each die's n_d pairs take units u = start + slot, start + slot + n_d, ... of
its contiguous range; all units have the same length, so the pairs run in
waves of n_d consecutive units. A unit is (m-block, split); inside an m-group
(group_m m-blocks) units are m-fastest, so the group_m units of one split are
consecutive. Assumption (the whole model): a split's W tiles are fetched
from DRAM once per wave that holds units of that split -- the units of a
split inside one wave walk its tiles in lockstep, so they share each fetch;
a later wave comes one unit duration (tps tiles) later, when the die has
streamed ~3 splits of other tiles (> the L2 left beside the resident A rows),
so it fetches again. A rows (evict_last) are fetched once.

    python scripts/k3_dram_model.py [--m 16384] [--v 126464] [--d 4096] [--pairs 37,37]
"""
from __future__ import annotations

import argparse
import math


def model(M: int, V: int, d: int, pairs: tuple[int, ...], group_m: int = 16, tps: int = 13) -> dict:
    m_blocks = math.ceil(M / 256)
    n_tiles = math.ceil(V / 256)
    S = math.ceil(n_tiles / tps)
    units = m_blocks * S
    tile_bytes = 256 * d * 2
    split_bytes = [min(tps, n_tiles - s * tps) * tile_bytes for s in range(S)]
    total_pairs = sum(pairs)
    # die ranges in proportion to the pairs (lmhead.cu: u0 = round(units * n0 / (n0 + n1)))
    bounds, acc = [0], 0
    for n in pairs:
        acc += n
        bounds.append(round(units * acc / total_pairs))

    def coords(u):
        per_group = group_m * S
        g, rem = divmod(u, per_group)
        gm = min(group_m, m_blocks - g * group_m)
        return g * group_m + rem % gm, rem // gm  # (m-block, split)

    w_bytes = 0
    for die, n in enumerate(pairs):
        lo, hi = bounds[die], bounds[die + 1]
        for w0 in range(lo, hi, n):
            fetched = set()
            for u in range(w0, min(w0 + n, hi)):
                mb, s = coords(u)
                key = (mb // group_m, s)  # a split's tiles, shared inside the wave by its m-group's units
                if key not in fetched:
                    fetched.add(key)
                    w_bytes += split_bytes[s]
    a_bytes = M * d * 2
    return {"m_blocks": m_blocks, "splits": S, "units": units, "w_bytes": w_bytes, "a_bytes": a_bytes,
            "dram_bytes": w_bytes + a_bytes, "w_reads": w_bytes / (n_tiles * tile_bytes),
            "floor_bytes": math.ceil(m_blocks / group_m) * n_tiles * tile_bytes + a_bytes}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--v", type=int, default=126464)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--pairs", default="37,37")
    ap.add_argument("--group-m", type=int, default=16)
    ap.add_argument("--tps", type=int, default=13)
    a = ap.parse_args()
    r = model(a.m, a.v, a.d, tuple(int(x) for x in a.pairs.split(",")), a.group_m, a.tps)
    print({k: (round(v / 1e9, 3) if k.endswith("bytes") else v) for k, v in r.items()})
