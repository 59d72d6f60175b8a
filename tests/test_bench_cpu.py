"""The reference arm of bench.py on CPU (-m "not gpu"): `bench.py --impl
reference` times the oracle on a bounded sample and prints one JSON line with
the contract's keys (impl, metric, value, unit, cpu_baseline, e2e, ...)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_oracle_sample_is_bounded_and_labelled():
    import bench
    r = bench.oracle_sample(0, seconds=0.5, omega=1.9)
    assert r["kind"] == "oracle" and r["cores"] == 1 and r["unit"] == "GNode-sweeps/s"
    assert r["value"] > 0 and "config0" in r["sample"]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "0", "--steps", "1", "--warmup", "0", "--ref-seconds", "1"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle"


# ------------------------------------------------- N > 1 transport check (gloo)
# bench.verify_p2p decides, on every rank identically, whether the peer-memory
# exchange fused into the sweep runs (its first window equals the NCCL
# transport's bit for bit on every rank) or NCCL does.  Its decision logic runs
# here with world size 2 over gloo and stand-in groups (no GPU).
class _FakeResult:
    def __init__(self, sweeps):
        self.sweeps = sweeps


class _FakeGroup:
    def __init__(self, V, sweeps, fail):
        self.V, self.sw, self.fail = V, sweeps, fail

    def transient(self, *a, **k):
        if self.fail:
            raise RuntimeError("watchdog: peer wait timed out")
        return _FakeResult(self.sw)

    def owned_voltages(self, g):
        return [(None, self.V)]

    def close(self):
        pass


def _verify_worker(rank, world, port, case, out):
    import numpy as np
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    V = np.linspace(0.9, 1.0, 12).reshape(3, 4) + rank
    sw = np.array([0, 6, 8, 8])

    def make_group(p2p=None, device=True):
        Vp, swp, fail = V.copy(), sw.copy(), False
        if p2p and case == "differ" and rank == 1:
            Vp[1, 2] = np.nextafter(Vp[1, 2], 2.0)          # one ulp on one rank
        if p2p and case == "counts" and rank == 0:
            swp[2] += 2
        if p2p and case == "raise":
            fail = True
        return _FakeGroup(Vp, swp, fail)

    class G:
        h = 5e-12

    out[rank] = bench.verify_p2p(None, G, rank, world, make_group, 4, 1e-10, 1.97)
    dist.destroy_process_group()


def _verify(case):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_verify_worker, args=(2, port, case, out), nprocs=2, join=True)
        return dict(out)


def test_verify_p2p_decision_world2():
    r = _verify("equal")
    assert r[0][0] is True and r[1][0] is True
    r = _verify("differ")                       # rank 1 differs: both ranks choose NCCL
    assert r[0][0] is False and r[1][0] is False
    assert "another rank" in r[0][1] and "differ" in r[1][1]
    r = _verify("counts")
    assert r[0][0] is False and r[1][0] is False
    r = _verify("raise")
    assert r[0][0] is False and r[1][0] is False and "raised" in r[0][1]
