"""The N > 1 decomposition path with real bricks on the GPU (decomposition.py:188-306).

Two ranks (gloo process group, both on cuda:0 -- functional coverage of the sharded code path on
a one-GPU box; the ranks never wait on each other's kernels) run train_decomposed on a 2x2x2
plan: rank r trains bricks flat % 2 == r.  In deterministic mode the bricks are byte-identical to
a one-rank run.  Each rank then holds only its own brick models and answers a query batch
through DecomposedField.forward_distributed (owner bucketing and row permutation in the library's
kernels, all-to-all over the group): every value equals the full field's."""
import json
import multiprocessing as mp
import os
import socket
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2308_02494_b200 as P  # noqa: E402
from paper_2308_02494_b200 import _lib as L  # noqa: E402
from paper_2308_02494_b200 import decomposition as D  # noqa: E402
from paper_2308_02494_b200 import model as PM  # noqa: E402
from paper_2308_02494_b200 import volume as PV  # noqa: E402

BLOB = [PV.BlobSpec(center=(0.2, -0.1, 0.3), sigma=(0.35, 0.3, 0.4)),
        PV.BlobSpec(center=(-0.4, 0.3, -0.2), sigma=(0.2, 0.25, 0.2), amplitude=0.5)]
MCFG = PM.ModelConfig(grids=8, channels=2, resolution=(6, 6, 6))
TCFG = dict(iterations=30, batch_size=512, delay_start=10, seed=5, plateau_enabled=False, deterministic=True)


def test_owner_bucket_and_permute_rows():
    rng = np.random.default_rng(3)
    for world, n in ((1, 10), (2, 1000), (5, 4097), (8, 0)):
        dest = rng.integers(0, world, n).astype(np.int64)
        perm, counts = D.owner_bucket(L.to_device(dest), world)
        p = L.to_host(perm)
        assert counts == np.bincount(dest, minlength=world).tolist()
        assert sorted(p.tolist()) == list(range(n))
        assert np.all(np.diff(dest[p]) >= 0)  # grouped by rank, rank 0 first
        x = rng.normal(size=(n, 3)).astype(np.float32)
        xd = L.to_device(x)
        g = D.permute_rows(xd, perm)
        assert np.array_equal(L.to_host(g), x[p])
        back = D.permute_rows(g, perm, scatter=True)
        assert np.array_equal(L.to_host(back), x)
    with pytest.raises(L.ApmgArgumentError, match="owner rank"):
        D.owner_bucket(L.to_device(np.array([0, 3], dtype=np.int64)), 2)


def _worker(rank, world, port, tmp, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tmp = Path(tmp)
        header = PV.load_header(tmp / "v.json")
        plan = P.plan_partition(header.dims, 2, 2, 2, ghost=1)
        man = P.train_decomposed(tmp / "v.raw", header, plan, MCFG, P.TrainConfig(**TCFG), tmp / "dist")
        full = P.DecomposedField.load(tmp / "dist" / "manifest.json")
        mine = P.DecomposedField(full.manifest, [m if b % world == rank else None for b, m in enumerate(full.models)])
        pts = np.random.default_rng(40 + rank).uniform(-1, 1, (3001 + 17 * rank, 3)).astype(np.float32)
        pd = L.to_device(pts)
        got = L.to_host(mine.forward_distributed(pd))
        want = L.to_host(full.forward_dev(pd))
        q.put((rank, [b.get("rank", None) for b in man.bricks], bool(np.array_equal(got, want)),
               float(np.max(np.abs(got - want)))))
    finally:
        dist.destroy_process_group()


def test_train_decomposed_two_ranks_real_bricks(tmp_path):
    vol = PV.synth_volume((20, 18, 16), BLOB)
    PV.save_volume(vol, tmp_path / "v.raw")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, _, ok, _ in res), res
    # one-rank run of the same plan: byte-identical bricks (deterministic mode), same manifest
    header = PV.load_header(tmp_path / "v.json")
    plan = P.plan_partition(header.dims, 2, 2, 2, ghost=1)
    P.train_decomposed(tmp_path / "v.raw", header, plan, MCFG, P.TrainConfig(**TCFG), tmp_path / "one")
    for b in range(8):
        assert (tmp_path / "dist" / f"brick_{b:04d}.apmg").read_bytes() == \
            (tmp_path / "one" / f"brick_{b:04d}.apmg").read_bytes(), b
    strip = ("train_seconds", "loop_ms")
    m2 = json.loads((tmp_path / "dist" / "manifest.json").read_text())
    m1 = json.loads((tmp_path / "one" / "manifest.json").read_text())
    for m in (m1, m2):
        for b in m["bricks"]:
            for k in strip:
                b.pop(k, None)
    assert m1 == m2
