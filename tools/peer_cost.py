"""Cost of the fused peer-memory exchanges (csrc/peer.cu, peer_gemv.cu) on one GPU.

Times, back to back with CUDA events (K launches per event pair):
  plain   cabl_cuda_dot                      (one kernel, no exchange)
  fused   cabl_cuda_dot_peer, world 1        (the same shard + publish/poll/sum)
  unfused cabl_cuda_dot(alpha0=0) + cabl_cuda_combine_partials  (the NCCL path minus NCCL)
for several n.  Prints one JSON line per n.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_02025_b200 as cb  # noqa: E402
from paper_2108_02025_b200 import _lib  # noqa: E402


def timed(fn, k=200, warm=10):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(k):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1000.0 / k


def main():
    L = _lib.lib()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    mb = C.c_void_p()
    _lib.call("cabl_peer_mailbox_create", C.byref(mb))
    tbl = (C.c_void_p * 1)(mb.value)
    for lg in (20, 24, 26, 28):
        n = 1 << lg
        x = cb.fill_uniform(torch.empty(n, device="cuda"), 1, 1)
        y = cb.fill_uniform(torch.empty(n, device="cuda"), 1, 2)
        out = torch.empty(1, device="cuda")
        parts = torch.empty(1, device="cuda")
        plain = lambda: L.cabl_cuda_dot_f32(x.data_ptr(), y.data_ptr(), n, 0.0, out.data_ptr(),  # noqa: E731
                                            8192, None, st)
        fused = lambda: L.cabl_cuda_dot_peer_f32(x.data_ptr(), y.data_ptr(), n, 0.0,  # noqa: E731
                                                 out.data_ptr(), tbl, 1, 0, 8192, None, st)

        def unfused():
            L.cabl_cuda_dot_f32(x.data_ptr(), y.data_ptr(), n, 0.0, parts.data_ptr(), 8192, None, st)
            L.cabl_cuda_combine_partials_f32(parts.data_ptr(), 1, 0.0, out.data_ptr(), st)
        r = {"n": n, "plain_us": timed(plain), "fused_us": timed(fused),
             "unfused_us": timed(unfused)}
        r = {k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}
        print(json.dumps(r), flush=True)
        del x, y
        torch.cuda.empty_cache()
    _lib.call("cabl_peer_mailbox_destroy", mb)

    # row-major GEMV: plain vs the gathering kernel at world 1 (c slice also
    # stored into the gathered buffer, completion words, epoch)
    for m, n in ((8192, 8192), (8192, 65536)):
        A = cb.fill_uniform(torch.empty(m * n, device="cuda"), 1, 3)
        x = cb.fill_uniform(torch.empty(n, device="cuda"), 1, 1)
        c = cb.fill_uniform(torch.empty(m, device="cuda"), 1, 4)
        buf, gmb = C.c_void_p(), C.c_void_p()
        _lib.call("cabl_peer_alloc", 2 * m * 4, C.byref(buf))
        _lib.call("cabl_peer_mailbox_create", C.byref(gmb))
        bt, mt = (C.c_void_p * 1)(buf.value), (C.c_void_p * 1)(gmb.value)
        plain = lambda: L.cabl_cuda_gemv_rm_f32(A.data_ptr(), m, n, x.data_ptr(), c.data_ptr(),  # noqa: E731
                                                8192, None, st)
        gath = lambda: L.cabl_cuda_gemv_rm_gather_f32(A.data_ptr(), m, n, x.data_ptr(),  # noqa: E731
                                                      c.data_ptr(), 0, m, bt, mt, 1, 0, None, st)
        r = {"gemv_m": m, "gemv_n": n, "plain_us": round(timed(plain), 2),
             "gather_us": round(timed(gath), 2)}
        print(json.dumps(r), flush=True)
        _lib.call("cabl_peer_free", buf)
        _lib.call("cabl_peer_mailbox_destroy", gmb)
        del A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
