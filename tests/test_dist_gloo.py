"""world_size-2 tests of the data-parallel plumbing on CPU (gloo backend).

The codec is rank-local; what crosses ranks is the max-over-ranks timing of
bench.py / train.py, rank 0's Adacc plan (broadcast, since every rank plans on
its own device profile), and DDP's gradient all-reduce.  The GPU runs use the
same code over NCCL.
"""

import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def gloo_results(tmp_path_factory):
    out = tmp_path_factory.mktemp("gloo")
    port = _free_port()
    procs = [subprocess.Popen([sys.executable, str(HERE / "_dist_worker.py"), str(r), "2", str(port), str(out)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for r in range(2)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=240)[0].decode(errors="replace"))
        except subprocess.TimeoutExpired:
            p.kill()
            pytest.fail("gloo worker timed out")
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [json.loads((out / f"rank{r}.json").read_text()) for r in range(2)]


def test_max_over_ranks_and_whole_job_rate(gloo_results):
    for res in gloo_results:
        assert res["max"] == 20.0
        assert res["rate_ms"] == 20.0
        assert res["rate"] == pytest.approx(2 * 1000.0 / 0.020)


def test_rank0_plan_is_broadcast(gloo_results):
    assert [r["agree_before"] for r in gloo_results] == [False, False]
    assert [r["agree_after"] for r in gloo_results] == [True, True]
    assert gloo_results[0]["plan"] == gloo_results[1]["plan"] == [[1, "retain"], [2, "compress"], [3, "retain"]]


def test_ddp_keeps_replicas_identical_on_different_batches(gloo_results):
    a, b = gloo_results
    assert a["batches_per_rank"][0] != a["batches_per_rank"][1]  # each rank sees its own data
    assert a["param_sums"][0] == a["param_sums"][1] == b["param_sums"][0]
    assert all(l == l and l < 20 for r in gloo_results for l in r["losses"])
