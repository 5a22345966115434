"""The slab exchange schedule (BASELINE configs[4]) without a GPU.

Both slab backends of libsrsb.so execute the SAME per-rank op lists (sr_sb_slab_schedule): the NCCL
backend as grouped ncclSend / ncclRecv on one GPU per process, the LOCAL backend (the single-GPU
emulation that tests/test_gpu_slab.py proves bitwise equal to one whole-image GPU run) as device
copies pairing the k-th send from r to d with the k-th receive on d from r.  Here the lists are
taken from the library on the CPU and

  * executed in one process with the LOCAL pairing rule on host buffers whose every element encodes
    its global (row, column) or (rank, index): the ghost rows / column segments must hold exactly
    the neighbours' rows / the transposed blocks (the layout the kernels read);
  * executed across 2 and 4 processes with torch.distributed gloo point-to-point (the message
    pairing of the NCCL path: every op of a rank posted, then all completed -- a group), and the
    result compared BITWISE with the in-process LOCAL execution.

A wrong offset, count, peer or phase order in the schedule fails one of them; a schedule that
pairs on one backend but not the other (a deadlock on NCCL) fails the cross-process run.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


@pytest.fixture(scope="module")
def S():
    from paper_2003_12693_b200 import build
    build.build()
    from paper_2003_12693_b200 import srsb
    return srsb


HALO_WRAP, HALO, A2A_FWD, A2A_BWD = 0, 1, 2, 3


# ----------------------------------------------------------------------------- host buffers
def _halo_buffers(P, Ml, gh, N):
    """Per rank: [(Ml + 2 gh) * N] float64, own rows = global row * N + column, ghosts NaN."""
    out = []
    for r in range(P):
        b = np.full(((Ml + 2 * gh) * N,), np.nan)
        rows = np.arange(r * Ml, (r + 1) * Ml)[:, None] * N + np.arange(N)[None, :]
        b[gh * N:(gh + Ml) * N] = rows.ravel()
        out.append({0: b})
    return out


def _a2a_buffers(P, Ml, N):
    """Per rank: buffer 0 (row-pass spectrum) and 1 (column buffer), 2 (N/2) Ml floats each."""
    n = N * Ml          # floats = 2 * (N/2) * Ml
    return [{0: r * 1e7 + np.arange(n, dtype=np.float64), 1: np.full((n,), np.nan)} for r in range(P)]


def _base(kind, gh, N):
    return gh * N if kind in (HALO_WRAP, HALO) else 0       # halo offsets are relative to local row 0


def _run_local(ops, bufs, kind, gh, N):
    """LOCAL pairing rule: the k-th send r -> d feeds the k-th receive on d from r."""
    P = len(ops)
    base = _base(kind, gh, N)
    recvq = {(d, s): [o for o in ops[d] if o[0] == 0 and o[1] == s] for d in range(P) for s in range(P)}
    used = {key: 0 for key in recvq}
    for r in range(P):
        for send, peer, buf, off, cnt in ops[r]:
            if not send:
                continue
            q = recvq[(peer, r)]
            k = used[(peer, r)]
            assert k < len(q), "a send without a matching receive"
            _, _, rbuf, roff, rcnt = q[k]
            used[(peer, r)] = k + 1
            assert rcnt == cnt
            bufs[peer][rbuf][base + roff:base + roff + cnt] = bufs[r][buf][base + off:base + off + cnt]
    assert all(used[k] == len(recvq[k]) for k in recvq), "a receive without a send"


def _schedule(S, kind, P, r, Ml, gh, N, k=0, nk=1):
    return S.slab_schedule(kind, P, r, Ml, gh, N, k, nk)


# ----------------------------------------------------------------------------- in-process checks
@pytest.mark.parametrize("P,Ml,gh,N", [(1, 16, 4, 32), (2, 16, 4, 32), (4, 8, 5, 16), (8, 8, 8, 64)])
@pytest.mark.parametrize("wrap", [True, False])
def test_halo_schedule_fills_the_neighbours_rows(S, P, Ml, gh, N, wrap):
    kind = HALO_WRAP if wrap else HALO
    ops = [_schedule(S, kind, P, r, Ml, gh, N) for r in range(P)]
    bufs = _halo_buffers(P, Ml, gh, N)
    _run_local(ops, bufs, kind, gh, N)
    M = P * Ml
    for r in range(P):
        b = bufs[r][0].reshape(Ml + 2 * gh, N)
        top, bot = b[:gh], b[gh + Ml:]
        cols = np.arange(N)[None, :]
        if r > 0 or wrap:                # rows r Ml - gh .. r Ml - 1 (periodic wrap at rank 0: Eq. 32)
            g = (np.arange(r * Ml - gh, r * Ml) % M)[:, None]
            assert np.array_equal(top, g * N + cols), r
        else:
            assert np.isnan(top).all()   # rank 0 without wrap: never written (Neumann rows, Q6)
        if r < P - 1 or wrap:
            g = (np.arange((r + 1) * Ml, (r + 1) * Ml + gh) % M)[:, None]
            assert np.array_equal(bot, g * N + cols), r
        else:
            assert np.isnan(bot).all()


@pytest.mark.parametrize("P,Ml,N,nk", [(1, 8, 16, 1), (2, 16, 32, 1), (2, 16, 32, 4), (4, 8, 64, 2),
                                       (8, 8, 128, 8), (8, 16, 64, 4)])
def test_alltoall_schedule_transposes_column_blocks(S, P, Ml, N, nk):
    """Forward: segment s of rank d's column buffer = block d of rank s's spectrum (all chunks);
    backward restores every spectrum exactly."""
    bufs = _a2a_buffers(P, Ml, N)
    orig = [b[0].copy() for b in bufs]
    blk = 2 * (N // 2 // P) * Ml          # floats per (src, dst) block
    for k in range(nk):
        _run_local([_schedule(S, A2A_FWD, P, r, Ml, 1, N, k, nk) for r in range(P)], bufs, A2A_FWD, 1, N)
    for d in range(P):
        for s in range(P):
            assert np.array_equal(bufs[d][1][s * blk:(s + 1) * blk], orig[s][d * blk:(d + 1) * blk]), (d, s)
    for b in bufs:
        b[0][:] = np.nan
    for k in range(nk):
        _run_local([_schedule(S, A2A_BWD, P, r, Ml, 1, N, k, nk) for r in range(P)], bufs, A2A_BWD, 1, N)
    for r in range(P):
        assert np.array_equal(bufs[r][0], orig[r])


def test_schedule_argument_errors(S):
    L = S.lib()
    assert L.sr_sb_slab_schedule(0, 2, 2, 8, 1, 16, 0, 1, None, 0) == -1        # rank out of range
    assert L.sr_sb_slab_schedule(2, 4, 0, 8, 1, 12, 0, 1, None, 0) == -1        # (N/2) % P != 0
    assert L.sr_sb_slab_schedule(2, 2, 0, 8, 1, 16, 0, 3, None, 0) == -1        # chunk does not divide
    assert L.sr_sb_slab_schedule(4, 2, 0, 8, 1, 16, 0, 1, None, 0) == -1        # bad kind
    assert L.sr_sb_slab_schedule(0, 1, 0, 8, 2, 16, 0, 1, None, 0) == 4         # P = 1: the wrap rows to self


# ----------------------------------------------------------------------------- across processes (gloo)
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [  # (kind, Ml, gh, N, nk)
    (HALO_WRAP, 16, 4, 32, 1), (HALO, 8, 5, 16, 1), (A2A_FWD, 16, 1, 64, 1), (A2A_FWD, 16, 1, 64, 4),
    (A2A_BWD, 8, 1, 32, 2),
]


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2003_12693_b200 import srsb as S
        results = []
        for kind, Ml, gh, N, nk in CASES:
            if kind in (HALO_WRAP, HALO):
                mine = _halo_buffers(world, Ml, gh, N)[rank]
            else:
                mine = _a2a_buffers(world, Ml, N)[rank]
                if kind == A2A_BWD:      # start from a filled column buffer
                    mine[1][:] = rank * 1e7 + 5e6 + np.arange(mine[1].size)
                    mine[0][:] = np.nan
            base = _base(kind, gh, N)
            t = {b: torch.from_numpy(v) for b, v in mine.items()}
            for k in range(nk):
                ops = S.slab_schedule(kind, world, rank, Ml, gh, N, k, nk)
                seq = {}                      # per-peer message number: the FIFO pairing as tags
                reqs, landing = [], []
                for send, peer, buf, off, cnt in ops:
                    key = (send, peer)
                    tag = seq.get(key, 0)
                    seq[key] = tag + 1
                    lo = base + off
                    if send:
                        if peer == rank:
                            landing.append(("self", tag, t[buf][lo:lo + cnt].clone()))
                        else:
                            reqs.append(dist.isend(t[buf][lo:lo + cnt].contiguous(), peer, tag=tag))
                    else:
                        if peer == rank:
                            landing.append(("selfrecv", tag, (buf, lo, cnt)))
                        else:
                            tmp = torch.empty(cnt, dtype=torch.float64)
                            reqs.append(dist.irecv(tmp, peer, tag=tag))
                            landing.append(("recv", tag, (buf, lo, cnt, tmp)))
                for r_ in reqs:
                    r_.wait()
                selfs = {tag: x for kind_, tag, x in landing if kind_ == "self"}
                for kind_, tag, x in landing:
                    if kind_ == "recv":
                        buf, lo, cnt, tmp = x
                        t[buf][lo:lo + cnt] = tmp
                    elif kind_ == "selfrecv":
                        buf, lo, cnt = x
                        t[buf][lo:lo + cnt] = selfs[tag]
            results.append({b: v.numpy().copy() for b, v in t.items()})
        q.put((rank, results))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_schedule_across_processes_matches_local_gloo(S, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=180) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for ci, (kind, Ml, gh, N, nk) in enumerate(CASES):
        if kind in (HALO_WRAP, HALO):
            bufs = _halo_buffers(world, Ml, gh, N)
        else:
            bufs = _a2a_buffers(world, Ml, N)
            if kind == A2A_BWD:
                for r in range(world):
                    bufs[r][1][:] = r * 1e7 + 5e6 + np.arange(bufs[r][1].size)
                    bufs[r][0][:] = np.nan
        for k in range(nk):
            _run_local([S.slab_schedule(kind, world, r, Ml, gh, N, k, nk) for r in range(world)], bufs, kind, gh, N)
        for r in range(world):
            for b in bufs[r]:
                a, ref = got[r][ci][b], bufs[r][b]
                assert np.array_equal(np.isnan(a), np.isnan(ref)) and np.array_equal(a[~np.isnan(a)], ref[~np.isnan(ref)]), \
                    (CASES[ci], r, b)
