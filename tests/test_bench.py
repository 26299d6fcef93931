"""Host-side checks of bench.py: the CPU arms' workload and timing plumbing, and
the --gpus N launch (re-exec under torch.distributed.run) with max-over-ranks
aggregation, exercised as world_size 2 over gloo on CPU."""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_cpu_shapes_match_the_gpu_workload():
    from paper_2508_00806_b200.workload import gpt_block_ops
    want = [(o.name, o.kind.value, o.rows, o.cols) for o in gpt_block_ops()]
    assert bench.block_shapes() == want


def test_cpu_sample_is_bf16_valued_and_deterministic():
    a = bench.cpu_sample(7, div=512)
    b = bench.cpu_sample(7, div=512)
    assert len(a) == 9
    for (ka, xa), (kb, xb) in zip(a, b):
        assert ka == kb and np.array_equal(xa, xb)
        if ka == "dropout_mask":
            assert xa.dtype == np.uint8 and set(np.unique(xa)) <= {0, 1}
        else:
            assert xa.dtype == np.float32
            assert not (xa.view(np.uint32) & 0xFFFF).any()  # bf16 values
            assert np.isfinite(xa).all()


def test_to_bf16_rounds_to_nearest_even():
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1.0 + 2 ** -9, -(1.0 + 2 ** -8 + 2 ** -20)], np.float32)
    got = bench._to_bf16_values(x)
    assert got.tolist() == [1.0, 1.0 + 2 ** -6, 1.0, -(1.0 + 2 ** -7)]


def test_cpu_pool_times_only_the_codec_loop():
    pool = bench.CpuPool(2, div=1024)
    try:
        gbs, wall, total = pool.measure(1)
    finally:
        pool.close()
    # bytes of both workers: each compresses+decompresses 9 tensors of >= 8 rows
    one = sum(2 * (x.size * (1 if k == "dropout_mask" else 2)) for k, x in bench.cpu_sample(0, 1024))
    assert total > 2 * one
    assert wall > 0 and gbs == total / wall / 1e9


def test_torchrun_command_line():
    cmd = bench.torchrun_argv(4, ["--gpus", "4", "--steps", "3"], 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:]


def test_gpus_2_launches_two_ranks_and_reports_max_over_ranks():
    """`python bench.py --gpus 2` (no WORLD_SIZE) re-execs as two ranks; rank r
    reports 10*(r+1) ms for 1 GB, so the whole-job rate is 2 GB / 20 ms."""
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dist-selftest"],
                         capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["ranks_env"] == "2"
    assert line["ms_max"] == 20.0
    assert line["value"] == 100.0
