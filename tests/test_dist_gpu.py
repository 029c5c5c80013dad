"""Two processes running the REAL kernels on one GPU (gloo for the
verification gather): each rank runs its shard of a fixed head set through
moba_attn forward + backward with no communication (dist.shard_fwd_bwd);
the gathered O / LSE / dQ / dK / dV equal a single-process run of all heads
bitwise (deterministic schedule). This is the code path bench.py takes
under torchrun on 2/4/8 GPUs."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

H, N, D, B, K = 6, 3072, 64, 128, 4


def _inputs():
    gen = torch.Generator(device="cuda").manual_seed(31)
    return [torch.randn(H, N, D, generator=gen, device="cuda").bfloat16() for _ in range(4)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_11571_b200 as mb
    from paper_2511_11571_b200 import _lib
    from paper_2511_11571_b200.dist import gather_and_compare, shard_fwd_bwd
    q, k, v, do = _inputs()
    n0 = _lib.load().moba_launch_count()
    (lo, hi), out, lse, dq, dk, dv = shard_fwd_bwd(q, k, v, do, B, K, rank, world, mode="tc", deterministic=True)
    launched = int(_lib.load().moba_launch_count() - n0)
    torch.cuda.synchronize()
    ref = None
    if rank == 0:
        xs = [t.clone().requires_grad_(True) for t in (q, k, v)]
        o, l = mb.moba_attn(*xs, B, K, mode="tc", deterministic=True, return_lse=True)
        o.backward(do)
        ref = {"O": o.detach().cpu(), "LSE": l.detach().cpu(), "dQ": xs[0].grad.cpu(), "dK": xs[1].grad.cpu(),
               "dV": xs[2].grad.cpu()}
    local = {"O": out.cpu(), "LSE": lse.cpu(), "dQ": dq.cpu(), "dK": dk.cpu(), "dV": dv.cpu()}
    res = gather_and_compare(local, ref, H, torch.device("cpu"))
    if rank == 0:
        torch.save({"res": res, "launched": launched}, os.path.join(out_dir, "res.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_share_gpu_gathered_equals_single():
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(2, _free_port(), tmp), nprocs=2, join=True)
        got = torch.load(os.path.join(tmp, "res.pt"))
    assert got["launched"] > 0          # the kernels ran in the rank processes
    for name, (bitwise, diff) in got["res"].items():
        assert bitwise, (name, diff)
