"""bench.py's multi-rank branch end to end (make the first 8-GPU
run low-risk): torchrun with 2, 4 and 8 ranks, vocab-sharded, both exchanges. Both
ranks share GPU 0 (MOSAIC_BENCH_SHARE_GPU=1) under a gloo group -- NCCL refuses
two ranks on one device -- so the NCCL-path code (all-gather of the triples +
rank-order merge) runs over gloo's all-gather and the p2p path (K4x peer
stores + signal pads) over torch symmetric memory mapped between the two
processes. The bench asserts inside that both ranks commit the identical
sequence with exactly k unmasked positions."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,exchange,e2e", [(2, "nccl", True), (2, "p2p", False), (4, "nccl", False),
                                                (4, "p2p", True), (8, "p2p", False)])
def test_bench_multi_rank(native_lib, world, exchange, e2e):
    """... and with e2e: each rank copies 1/N of H's rows from the host and the
    all-gather assembles the rest (bench.py asserts every rank's H equals the
    generated one and the read-back x is the committed step)."""
    env = {**os.environ, "MOSAIC_BENCH_SHARE_GPU": "1"}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", str(world),
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-activation",
           "--backend", "gloo", "--exchange", exchange] + ([] if e2e else ["--no-e2e"])
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 prints the one line
    line = lines[0]
    assert line["n_gpus"] == world and line["value"] > 0 and line["config"]["vocab_shard"] == 126464 // world
    assert exchange in line["config"]["parallelism"]
    assert line["gpu_launches"] > 0
    if e2e:
        assert line["e2e"]["value"] > 0
        assert line["e2e"]["h2d_bytes_per_step"] == 32768 * 4 + 32768 // world * 4096 * 2
