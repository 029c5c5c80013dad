"""Varlen (build_varlen) timing and bitwise check on tc-router plans.

usage: python scripts/varlen_probe.py [N ...]   (32 heads, d=64, B=128, top-k 8)
Times moba_varlen alone (CUDA events, 20 launches) for each N and checks
flat / row_pos / counts / offsets against a torch.sort of the (block, query)
pairs.
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device, _lib  # noqa: E402


def reference_plan(topk, n):
    H, N, W = topk.shape
    out = []
    for h in range(H):
        t = topk[h].reshape(-1).long()
        q = torch.arange(N, device=t.device).repeat_interleave(W)
        ok = t >= 0
        key = torch.where(ok, t * N + q, torch.full_like(t, 1 << 62))
        srt, perm = torch.sort(key, stable=True)
        nv = int(ok.sum())
        flat = (srt[:nv] % N).int()
        rp = torch.full_like(t, -1)
        rp[perm[:nv]] = torch.arange(nv, device=t.device)
        counts = torch.bincount(t[ok], minlength=n).int()
        out.append((flat, rp.view(N, W).int(), counts))
    return out


def main():
    Ns = [int(x) for x in sys.argv[1:]] or [8192, 65536, 262144, 524288]
    lib = _lib.load()
    H, D, B, K = 32, 64, 128, 8
    torch.manual_seed(0)
    for N in Ns:
        n = -(-N // B)
        q = torch.randn(H, N, D, device="cuda", dtype=torch.bfloat16)
        cent = torch.randn(H, n, D, device="cuda", dtype=torch.float32)
        plan = _device.route(q, cent, B, K, mode=_lib.MOBA_ROUTE_TC)
        topk = plan.topk
        del q
        W = K + 1
        ref = reference_plan(topk, n) if N <= 262144 else None
        ws = torch.empty(lib.moba_route_workspace_size(H, N, B, K), dtype=torch.uint8, device="cuda")
        counts = torch.empty(H, n, dtype=torch.int32, device="cuda")
        offsets = torch.empty_like(counts)
        flat = torch.empty(H, N * W, dtype=torch.int32, device="cuda")
        row_pos = torch.empty(H, N, W, dtype=torch.int32, device="cuda")
        s = torch.cuda.current_stream().cuda_stream

        def run():
            st = lib.moba_varlen(topk.data_ptr(), H, N, W, B, counts.data_ptr(), offsets.data_ptr(),
                                 flat.data_ptr(), row_pos.data_ptr(), ws.data_ptr(), ws.numel(), s)
            _lib.check(st, "moba_varlen")

        for _rep in range(1):
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            ok = "unchecked"
            if ref is not None:
                ok = "bitwise-ok"
                for h in range(H):
                    rf, rr, rc = ref[h]
                    nv = rf.numel()
                    if not (torch.equal(flat[h, :nv], rf) and torch.equal(row_pos[h], rr)
                            and torch.equal(counts[h], rc)):
                        ok = f"MISMATCH head {h}"
                        break
                    if not torch.equal(offsets[h], torch.cumsum(rc, 0).int() - rc):
                        ok = f"MISMATCH offsets head {h}"
                        break
            print(f"N={N} varlen {ms:.4f} ms  {ok}", flush=True)


if __name__ == "__main__":
    main()
