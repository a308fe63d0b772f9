"""Multi-GPU partition and exchange logic of paper_2108_02025_b200.shard,
exercised as 2 (and 3) CPU processes over gloo — the same collectives the GPU
ranks issue over NCCL, with the per-rank compute injected (the oracle as the
local op, a rank-ordered numpy sum as the combine).  The GPU build only ever
runs one GPU here, so this is where the N > 1 host path is tested.

Checks: balanced contiguous partition; sharded DOT = rank-ordered sum of the
shard partials + alpha0 (bitwise, identical on every rank, independent of
which rank finishes first); row-sharded GEMV with gather reproduces the
single-process oracle bitwise (rows are independent); row-sharded GER needs no
communication and reproduces the oracle bitwise; the peer-DOT mailbox exchange
(IPC handles all-gathered, peers imported) builds every rank's pointer table
in rank order.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2108_02025_b200 import shard


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ordered_combine(gathered: torch.Tensor, alpha0: float, out: torch.Tensor) -> None:
    dt = gathered.numpy().dtype.type
    total = dt(0)
    for p in gathered.numpy():
        total = dt(total + p)
    out[0] = torch.tensor(dt(total + dt(alpha0)))


def _oracle_partial(x, y, out, policy):
    out[0] = torch.tensor(O.dot_ref(x.numpy(), y.numpy(), 0.0))


def _oracle_gemv_rows(A, x, c, policy):
    cn = c.numpy()
    O.gemv_ref(A.data.numpy(), int(A.layout()), x.numpy(), cn)


def _oracle_ger(x, y, C, policy):
    O.ger_ref(x.numpy(), y.numpy(), C.data.numpy(), int(C.layout()))


def _oracle_gemv_cols(A, x, c, policy):
    O.gemv_ref(A.data.numpy(), int(A.layout()), x.numpy(), c.numpy())


def _ordered_combine_rows(parts: torch.Tensor, world: int, c: torch.Tensor) -> None:
    P = parts.numpy().reshape(world, -1)
    dt = P.dtype.type
    total = np.zeros(P.shape[1], dtype=P.dtype)
    for g in range(world):
        total = (total + P[g]).astype(P.dtype)
    c.copy_(torch.from_numpy((c.numpy() + total).astype(P.dtype)))
    assert dt is not None


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2108_02025_b200 as cb
    pol = cb.default_policy(1)
    try:
        # ---- DOT: chunk-sharded, all-gather of partials, ordered combine
        n = 100_003
        for dt in (np.float32, np.float64):
            x = O.gen_uniform(n, dt, 42, 1)
            y = O.gen_uniform(n, dt, 42, 2)
            b, e = shard.partition(n, world, rank)
            out = torch.zeros(1, dtype=torch.from_numpy(x).dtype)
            shard.sharded_dot(torch.from_numpy(x[b:e].copy()), torch.from_numpy(y[b:e].copy()),
                              0.75, out, pol, partial_fn=_oracle_partial,
                              combine_fn=_ordered_combine)
            results[f"dot_{np.dtype(dt).name}_{rank}"] = float(out[0])
        # ---- DOT with a GPU-count-invariant result: fixed global segments
        ni, seg = 100_003, 4096  # 25 segments, the last one ragged
        for dt in (np.float32, np.float64):
            x = O.gen_uniform(ni, dt, 42, 1)
            y = O.gen_uniform(ni, dt, 42, 2)
            b, e = shard.invariant_range(ni, seg, world, rank)
            out = torch.zeros(1, dtype=torch.from_numpy(x).dtype)
            shard.sharded_dot_invariant(torch.from_numpy(x[b:e].copy()),
                                        torch.from_numpy(y[b:e].copy()), 0.75, out, pol,
                                        n_total=ni, segment=seg, partial_fn=_oracle_partial,
                                        combine_fn=_ordered_combine)
            results[f"doti_{np.dtype(dt).name}_{rank}"] = float(out[0])
        # ---- GEMV row blocks + gather
        m, k = 1001, 257
        A = O.gen_uniform(m * k, np.float64, 42, 3).reshape(m, k)
        xv = O.gen_uniform(k, np.float64, 42, 1)
        c0 = O.gen_uniform(m, np.float64, 42, 4)
        b, e = shard.partition(m, world, rank)
        Aloc = cb.DenseMatrix.wrap(torch.from_numpy(A[b:e].reshape(-1).copy()), e - b, k,
                                   cb.Layout.RowMajor)
        cloc = torch.from_numpy(c0[b:e].copy())
        full = shard.sharded_gemv_rows(Aloc, torch.from_numpy(xv), cloc, pol, gather=True,
                                       m_total=m, local_fn=_oracle_gemv_rows)
        results[f"gemv_{rank}"] = full.numpy().copy()
        # equal slices gathered straight into a caller-owned result (m = 1002 = 2 * 3 * 167)
        me = 1002
        Ae = O.gen_uniform(me * k, np.float64, 42, 3).reshape(me, k)
        ce = O.gen_uniform(me, np.float64, 42, 4)
        b2, e2 = shard.partition(me, world, rank)
        Ae_loc = cb.DenseMatrix.wrap(torch.from_numpy(Ae[b2:e2].reshape(-1).copy()), e2 - b2, k,
                                     cb.Layout.RowMajor)
        dest = torch.full((me,), float("nan"), dtype=torch.float64)
        got = shard.sharded_gemv_rows(Ae_loc, torch.from_numpy(xv), torch.from_numpy(ce[b2:e2].copy()),
                                      pol, gather=True, m_total=me, local_fn=_oracle_gemv_rows,
                                      out=dest)
        assert got is dest
        results[f"gemv_even_{rank}"] = dest.numpy().copy()
        # ragged slices into a caller-owned result too
        dest2 = torch.full((m,), float("nan"), dtype=torch.float64)
        shard.sharded_gemv_rows(Aloc, torch.from_numpy(xv), torch.from_numpy(c0[b:e].copy()), pol,
                                gather=True, m_total=m, local_fn=_oracle_gemv_rows, out=dest2)
        results[f"gemv_out_{rank}"] = dest2.numpy().copy()
        # ---- GER row blocks, no communication
        gx = O.gen_uniform(m, np.float32, 42, 1)
        gy = O.gen_uniform(k, np.float32, 42, 2)
        C0 = O.gen_uniform(m * k, np.float32, 42, 5).reshape(m, k)
        Cloc = cb.DenseMatrix.wrap(torch.from_numpy(C0[b:e].reshape(-1).copy()), e - b, k,
                                   cb.Layout.RowMajor)
        shard.sharded_ger_rows(torch.from_numpy(gx[b:e].copy()), torch.from_numpy(gy), Cloc, pol,
                               local_fn=_oracle_ger)
        results[f"ger_{rank}"] = (b, e, Cloc.data.numpy().copy())
        # ---- col-major GEMV by column blocks, all-gather + rank-ordered combine
        mc, kc = 64, 5003
        Ac = O.gen_uniform(mc * kc, np.float64, 42, 6)  # col-major: column j at j*mc
        xc = O.gen_uniform(kc, np.float64, 42, 7)
        cc = O.gen_uniform(mc, np.float64, 42, 8)
        b, e = shard.partition(kc, world, rank)
        Aloc = cb.DenseMatrix.wrap(torch.from_numpy(Ac[b * mc:e * mc].copy()), mc, e - b,
                                   cb.Layout.ColMajor)
        cl = torch.from_numpy(cc.copy())
        shard.sharded_gemv_cols(Aloc, torch.from_numpy(xc[b:e].copy()), cl, pol,
                                local_fn=_oracle_gemv_cols, combine_fn=_ordered_combine_rows)
        results[f"gemvcols_{rank}"] = cl.numpy().copy()
        # ---- peer-DOT mailboxes: IPC handles all-gathered, peers imported,
        # the pointer table in rank order with this rank's own mailbox at [rank]
        mb = shard.PeerMailboxes(torch.device("cpu"), create=lambda: 1000 + rank,
                                 export=lambda p: f"h{p}".encode().ljust(64, b"\0"),
                                 import_=lambda h: 2000 + int(h.rstrip(b"\0")[1:]))
        results[f"peer_{rank}"] = (mb.world, mb.rank, [mb.table[g] for g in range(world)])
        # gathered-GEMV buffers: (buffer, mailbox) handles exchanged in one
        # all-gather, both tables in rank order
        gg = shard.GatherGemv(torch.device("cpu"), 100, torch.float32,
                              alloc=lambda nb: 5000 + rank, create=lambda: 6000 + rank,
                              export=lambda p: f"h{p}".encode().ljust(64, b"\0"),
                              import_=lambda h: 10000 + int(h.rstrip(b"\0")[1:]))
        results[f"gg_{rank}"] = ([gg.cfull_table[g] for g in range(world)],
                                 [gg.mbox_table[g] for g in range(world)])
        pr = shard.PeerRows(torch.device("cpu"), 64, torch.float64,
                            alloc=lambda nb: 7000 + rank, create=lambda: 8000 + rank,
                            export=lambda p: f"h{p}".encode().ljust(64, b"\0"),
                            import_=lambda h: 10000 + int(h.rstrip(b"\0")[1:]))
        results[f"pr_{rank}"] = ([pr.slot_table[g] for g in range(world)],
                                 [pr.mbox_table[g] for g in range(world)])
        # an import failure on one rank is reported on every rank (no rank may
        # go on to spin on a peer that never arrives)
        def bad_import(h):
            if rank == world - 1:
                raise OSError("no IPC here")
            return 1
        try:
            shard.PeerMailboxes(torch.device("cpu"), create=lambda: 1, export=lambda p: b"h",
                                import_=bad_import)
            results[f"peerfail_{rank}"] = "no error"
        except RuntimeError as e:
            results[f"peerfail_{rank}"] = str(e)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_paths_over_gloo(world):
    O.lib()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)

    # DOT: every rank holds the same value = ordered sum of shard partials + alpha0
    n = 100_003
    for dt in (np.float32, np.float64):
        x, y = O.gen_uniform(n, dt, 42, 1), O.gen_uniform(n, dt, 42, 2)
        total = dt(0)
        for r in range(world):
            b, e = shard.partition(n, world, r)
            total = dt(total + O.dot_ref(x[b:e], y[b:e], 0.0))
        want = float(dt(total + dt(0.75)))
        got = {results[f"dot_{np.dtype(dt).name}_{r}"] for r in range(world)}
        assert got == {want}
        # and it agrees with the single-process oracle within the contract bound
        truth, sumabs = O.dot_truth(x, y, 0.75)
        assert abs(want - truth) <= 4 * n * np.finfo(dt).eps * (sumabs + 0.75)

    # invariant DOT: the segment partials summed in index order — the same value for
    # every world size (computed here with no process group at all, i.e. one rank)
    ni, seg = 100_003, 4096
    for dt in (np.float32, np.float64):
        x, y = O.gen_uniform(ni, dt, 42, 1), O.gen_uniform(ni, dt, 42, 2)
        total = dt(0)
        for k in range(0, ni, seg):
            total = dt(total + O.dot_ref(x[k:k + seg], y[k:k + seg], 0.0))
        want = float(dt(total + dt(0.75)))
        got = {results[f"doti_{np.dtype(dt).name}_{r}"] for r in range(world)}
        assert got == {want}
        import paper_2108_02025_b200 as cb
        one = torch.zeros(1, dtype=torch.from_numpy(x).dtype)
        shard.sharded_dot_invariant(torch.from_numpy(x), torch.from_numpy(y), 0.75, one,
                                    cb.default_policy(1), n_total=ni, segment=seg,
                                    partial_fn=_oracle_partial, combine_fn=_ordered_combine)
        assert float(one[0]) == want

    # GEMV: gathered c equals the single-process oracle bitwise on every rank
    m, k = 1001, 257
    A = O.gen_uniform(m * k, np.float64, 42, 3)
    xv = O.gen_uniform(k, np.float64, 42, 1)
    c = O.gen_uniform(m, np.float64, 42, 4)
    O.gemv_ref(A, 0, xv, c)
    for r in range(world):
        np.testing.assert_array_equal(results[f"gemv_{r}"], c)
        np.testing.assert_array_equal(results[f"gemv_out_{r}"], c)
    me = 1002
    Ae = O.gen_uniform(me * k, np.float64, 42, 3)
    ce = O.gen_uniform(me, np.float64, 42, 4)
    O.gemv_ref(Ae, 0, xv, ce)
    for r in range(world):
        np.testing.assert_array_equal(results[f"gemv_even_{r}"], ce)

    # GER: the row blocks tile C and match the oracle bitwise
    gx, gy = O.gen_uniform(m, np.float32, 42, 1), O.gen_uniform(k, np.float32, 42, 2)
    C = O.gen_uniform(m * k, np.float32, 42, 5)
    O.ger_ref(gx, gy, C, 0)
    C = C.reshape(m, k)
    covered = 0
    for r in range(world):
        b, e, blk = results[f"ger_{r}"]
        np.testing.assert_array_equal(blk.reshape(e - b, k), C[b:e])
        covered += e - b
    assert covered == m

    # col-major GEMV by columns: c + sum over ranks (rank order) of the column
    # blocks' partials, identical on every rank
    mc, kc = 64, 5003
    Ac = O.gen_uniform(mc * kc, np.float64, 42, 6)
    xc = O.gen_uniform(kc, np.float64, 42, 7)
    cc = O.gen_uniform(mc, np.float64, 42, 8)
    total = np.zeros(mc)
    for r in range(world):
        b, e = shard.partition(kc, world, r)
        part = np.zeros(mc)
        O.gemv_ref(Ac[b * mc:e * mc].copy(), 1, xc[b:e].copy(), part)
        total = total + part
    want = cc + total
    for r in range(world):
        np.testing.assert_array_equal(results[f"gemvcols_{r}"], want)
    truth, rowabs = O.gemv_truth(Ac, 1, xc, cc)
    assert np.all(np.abs(want - truth) <= 4 * kc * np.finfo(np.float64).eps * (rowabs + np.abs(cc)))


    # peer-DOT mailbox tables: own mailbox at [rank], rank g's import elsewhere
    for r in range(world):
        w, rk, table = results[f"peer_{r}"]
        assert (w, rk) == (world, r)
        assert table == [1000 + r if g == r else 2000 + 1000 + g for g in range(world)]
        assert results[f"peerfail_{r}"].startswith("peer mailbox exchange failed")
        bufs, mbs = results[f"gg_{r}"]
        assert bufs == [5000 + r if g == r else 15000 + g for g in range(world)]
        assert mbs == [6000 + r if g == r else 16000 + g for g in range(world)]
        slots, mbs = results[f"pr_{r}"]
        assert slots == [7000 + r if g == r else 17000 + g for g in range(world)]
        assert mbs == [8000 + r if g == r else 18000 + g for g in range(world)]


def test_partition_is_balanced_and_contiguous():
    for total in (0, 1, 7, 8192, 65536, 100_003, 1 << 32):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.partition(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
