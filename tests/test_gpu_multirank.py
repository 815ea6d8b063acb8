"""Multi-rank paths on one GPU: the ranks run with the gloo backend
(PGSAG_DIST_BACKEND=gloo: host collectives, every rank on cuda:0).  No kernel of one rank waits
on another rank's, so this checks the sharding and the collectives' results, not performance.

- §8(e): every sub-region's outputs under the 2-rank strong-scaling layout (each rank owns 4 of
  the 8 C4 sub-regions) equal its 1-rank outputs: forward images bit-identical (A6 is
  deterministic), entry counts equal, gradient sums within float32 atomic-order rounding.
- NEXT-4 (not in the paper, P:51 trains groups independently): two ranks sharing one sub-region
  average their gradients each iteration (shard.allreduce_mean) and sum the densification
  statistics; after training with densification both members hold bit-identical parameters
  and Adam moments.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(cmd, nproc, timeout=900):
    env = dict(os.environ, PGSAG_DIST_BACKEND="gloo")
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", f"--master-port={_port()}"] + cmd
    else:
        cmd = [sys.executable] + cmd
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r.stdout


def test_subregions_equal_one_vs_two_ranks(tmp_path):
    args = ["bench.py", "--config", "c4", "--n-gaussians", "20000", "--image", "960x640", "--steps", "2",
            "--warmup", "1", "--no-cpu", "--no-e2e", "--no-train"]
    one, two = tmp_path / "one.json", tmp_path / "two.json"
    l1 = json.loads(_run(args + ["--digests", str(one)], 1).strip().splitlines()[-1])
    l2 = json.loads(_run(args + ["--gpus", "2", "--digests", str(two)], 2).strip().splitlines()[-1])
    assert l1["scaling"] == "strong" and l2["n_gpus"] == 2 and l2["config"]["views_per_step"] == 8
    a = {(d["region"], d["view"]): d for d in json.load(open(one))}
    b = {(d["region"], d["view"]): d for d in json.load(open(two))}
    assert set(a) == set(b) and {k[0] for k in a} == set(range(8))
    for k in a:
        assert a[k]["M"] == b[k]["M"], k
        assert a[k]["fwd"] == b[k]["fwd"], k
        for c, x in a[k]["grad_sums"].items():
            y = b[k]["grad_sums"][c]
            assert abs(x - y) <= 1e-5 * max(abs(x), 1e-30), (k, c, x, y)


def test_view_parallel_members_stay_identical():
    out = _run(["-m", "paper_2501_01677_b200.groups", "--regions", "1", "--small", "--iters", "6",
                "--densify-every", "3", "--views", "4"], 2)
    rep = json.loads(out.strip().splitlines()[-1])
    rs = [x for x in rep["reports"] if x["region"] == 0]
    assert len(rs) == 2 and {x["dp_rank"] for x in rs} == {0, 1} and all(x["dp_size"] == 2 for x in rs)
    assert rs[0]["state_digest"] == rs[1]["state_digest"]
    assert rs[0]["n_gaussians"] == rs[1]["n_gaussians"]
    # the members trained different views: their last photometric losses differ
    assert rs[0]["final_loss"]["rgb"] != rs[1]["final_loss"]["rgb"]
