"""Multi-GPU partition logic on the CPU (no GPU needed): the rank plans of host/distribute.cpp
reproduce the single-process sums exactly.

The reference's cross-subdomain sums are serial loops in ascending subdomain order
(src/preconditioner.cpp:141-147 r_c, :168-169 / :189-190 prolongation, src/csr_matrix.cpp:90-102
SpMV). Here every rank holds a block of subdomains; with the plan's halo and interface exchanges
(run through torch.distributed gloo with world_size 2, and simulated in-process for 4 and 8
ranks) the distributed SpMV, the owner-ordered interface sums and the gathered coarse residual
must equal the global computation BIT FOR BIT, and the owned sets must partition the dofs.
"""
import os
import socket

import numpy as np
import pytest

from paper_2410_14786_b200 import Problem, RankPlan


def _csr(t):
    nr, nc, rp, ci, va = t
    return nr, nc, rp, ci, va


def spmv_rows(csr, x, rows):
    nr, nc, rp, ci, va = csr
    y = np.zeros(len(rows))
    for k, i in enumerate(rows):
        acc = 0.0
        for p in range(rp[i], rp[i + 1]):  # row-sequential in stored column order
            acc += va[p] * x[ci[p]]
        y[k] = acc
    return y


def global_iface_sum(prob, h_of):
    """z[g] = sum over subdomains containing g (ascending) of h_j[g], interface dofs only."""
    dofs, ni = prob.subdomain_dofs(), prob.interior_counts()
    z = {}
    for j in range(prob.n_subdomains):
        for g in dofs[j][ni[j]:]:
            z[int(g)] = z.get(int(g), 0.0) + h_of(j, int(g))
    return z


def h_value(j, g):
    return np.sin(0.37 * j + 0.011 * g) * (1.0 + j)


def plan_checks(prob, world, exchange):
    """Run the checks for all ranks; `exchange(plans, rank, send_lists)` returns what each rank
    receives from each peer (list per peer, in the peer order of the plan)."""
    n = prob.global_dofs
    plans = [RankPlan(prob, r, world) for r in range(world)]
    # owned sets partition the dofs; rows = dofs of the rank's subdomains
    owned = np.concatenate([p.local_to_global[:p.n_owned] for p in plans])
    assert np.array_equal(np.sort(owned), np.arange(n))
    dofs = prob.subdomain_dofs()
    for p in plans:
        mine = np.unique(np.concatenate([dofs[j] for j in p.subdomains]))
        assert np.array_equal(np.sort(p.local_to_global[:p.n_rows]), mine)
        lp = p.local_problem
        for li, j in enumerate(p.subdomains):
            assert np.array_equal(p.local_to_global[lp.subdomain_dofs()[li]], dofs[j])
            a, b = lp.local_matrix(li), prob.local_matrix(j)
            assert all(np.array_equal(u, v) for u, v in zip(a[2:], b[2:]))
    # distributed SpMV with the halo exchange == global SpMV (bitwise)
    A = prob.global_matrix()
    x = np.cos(np.arange(n) * 0.013) + 0.5
    yg = spmv_rows(A, x, range(n))
    sends = []
    for p in plans:
        xl = np.zeros(p.n_local)
        xl[:p.n_rows] = x[p.local_to_global[:p.n_rows]]
        sends.append([xl[p.halo_send_idx[p.halo_send_off[k]:p.halo_send_off[k + 1]]] for k in range(len(p.halo_peers))])
    recv = exchange(plans, "halo", sends)
    for r, p in enumerate(plans):
        xl = np.zeros(p.n_local)
        xl[:p.n_rows] = x[p.local_to_global[:p.n_rows]]
        for k in range(len(p.halo_peers)):
            xl[p.n_rows + p.halo_recv_off[k]:p.n_rows + p.halo_recv_off[k + 1]] = recv[r][k]
        assert np.array_equal(xl, x[p.local_to_global])
        y = spmv_rows(p.local_problem.global_matrix(), xl, range(p.n_rows))
        assert np.array_equal(y, yg[p.local_to_global[:p.n_rows]])
    # interface sums through local + remote slots in ascending subdomain order == global
    zg = global_iface_sum(prob, h_value)
    ni = prob.interior_counts()
    sends, slots_all = [], []
    for p in plans:
        slots = []  # local slot -> (global subdomain, global dof), subdomain-major
        for j in p.subdomains:
            slots += [(int(j), int(g)) for g in dofs[j][ni[j]:]]
        assert len(slots) == p.n_local_slots
        slots_all.append(slots)
        hv = np.array([h_value(j, g) for j, g in slots])
        sends.append([hv[p.iface_send_slot[p.iface_send_off[k]:p.iface_send_off[k + 1]]]
                      for k in range(len(p.iface_peers))])
    recv = exchange(plans, "iface", sends)
    for r, p in enumerate(plans):
        remote = np.zeros(p.n_remote_slots)
        for k in range(len(p.iface_peers)):
            remote[p.iface_recv_off[k]:p.iface_recv_off[k + 1]] = recv[r][k]
        g2l = {int(g): l for l, g in enumerate(p.local_to_global)}
        owners = {}
        for s, (j, g) in enumerate(slots_all[r]):
            owners.setdefault(g2l[g], []).append((j, h_value(j, g)))
        for l in range(p.n_rows):
            for e in range(p.remote_ptr[l], p.remote_ptr[l + 1]):
                owners.setdefault(l, []).append((int(p.remote_subdomain[e]), remote[p.remote_slot[e]]))
        for l, lst in owners.items():
            acc = 0.0
            for _, v in sorted(lst, key=lambda t: t[0]):
                acc += v
            assert acc == zg[int(p.local_to_global[l])]
    # gathered coarse contributions: every subdomain at cbuf_offset, padded per rank
    prim = prob.primal_maps()
    pad = plans[0].cbuf_pad
    for p in plans:
        assert p.cbuf_pad == pad and np.array_equal(p.cbuf_offset, plans[0].cbuf_offset)
        for j in p.subdomains:
            assert p.rank * pad <= p.cbuf_offset[j] and p.cbuf_offset[j] + len(prim[j]) <= (p.rank + 1) * pad
    return plans


def local_exchange(plans, kind, sends):
    """In-process stand-in for the grouped ncclSend/ncclRecv of device/comm.cu."""
    peers = {r: list(p.halo_peers if kind == "halo" else p.iface_peers) for r, p in enumerate(plans)}
    out = []
    for r, p in enumerate(plans):
        got = []
        for q in peers[r]:
            got.append(sends[q][peers[q].index(r)])
        out.append(got)
    return out


@pytest.mark.parametrize("cells,k,world", [((32, 16), (4, 2), 2), ((32, 32), (4, 4), 4), ((64, 32), (8, 4), 8),
                                           ((24, 24), (3, 3), 3)])
def test_rank_plans_reproduce_global_sums(cells, k, world):
    prob = Problem.poisson(cells[0], k[0], cells[1], k[1])
    plans = plan_checks(prob, world, local_exchange)
    if k == (4, 4) and world == 4:  # 2x2 rectangular blocks of 2x2 subdomains
        assert sorted(len(p.subdomains) for p in plans) == [4, 4, 4, 4]
        assert all(len(p.halo_peers) == 3 for p in plans)  # edge + edge + diagonal neighbour


def test_c2_layout_blocks():
    # C2 weak scaling: 64 subdomains per rank as 8x8 blocks
    prob = Problem.poisson(64, 16, 32, 8)  # 16x8 layout, m=4
    plans = [RankPlan(prob, r, 2) for r in range(2)]
    for p in plans:
        assert len(p.subdomains) == 64
        sx = set(int(j) % 16 for j in p.subdomains)
        assert len(sx) == 8


def test_bad_partitions_rejected():
    prob = Problem.poisson(16, 2)
    with pytest.raises(ValueError):
        RankPlan(prob, 0, 8)  # more ranks than subdomains
    with pytest.raises(ValueError):
        RankPlan(prob, 0, 2, subdomain_rank=[0, 0, 0, 0])  # rank 1 owns nothing


# ---- world_size 2 over torch.distributed gloo (real processes)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, result_dir):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    prob = Problem.poisson(32, 4, 16, 2)

    def gloo_exchange(plans, kind, sends):
        # only this rank's lists are real; exchange them with the peers over gloo
        p = plans[rank]
        peers = list(p.halo_peers if kind == "halo" else p.iface_peers)
        got = []
        for k, q in enumerate(peers):
            buf = torch.from_numpy(np.ascontiguousarray(sends[rank][k]))
            n_recv = (p.halo_recv_off[k + 1] - p.halo_recv_off[k]) if kind == "halo" else (
                p.iface_recv_off[k + 1] - p.iface_recv_off[k])
            rbuf = torch.zeros(int(n_recv), dtype=torch.float64)
            if rank < q:
                dist.send(buf, q)
                dist.recv(rbuf, q)
            else:
                dist.recv(rbuf, q)
                dist.send(buf, q)
            got.append(rbuf.numpy())
        out = [None] * world
        out[rank] = got
        # the other rank's checks run in its own process: feed it the true lists locally
        for r in range(world):
            if r != rank:
                out[r] = local_exchange(plans, kind, sends)[r]
        return out

    plan_checks(prob, world, gloo_exchange)
    # coarse: allgather of padded per-rank blocks reproduces the global r_c order
    plan = RankPlan(prob, rank, world)
    prim = prob.primal_maps()
    cb = torch.zeros(world * plan.cbuf_pad, dtype=torch.float64)
    for j in plan.subdomains:
        for t in range(len(prim[j])):
            cb[plan.cbuf_offset[j] + t] = float(j * 10 + t)
    parts = [torch.zeros(plan.cbuf_pad, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, cb[rank * plan.cbuf_pad:(rank + 1) * plan.cbuf_pad].clone())
    full = torch.cat(parts).numpy()
    for j in range(prob.n_subdomains):
        for t in range(len(prim[j])):
            assert full[plan.cbuf_offset[j] + t] == float(j * 10 + t)
    open(os.path.join(result_dir, f"ok{rank}"), "w").write("ok")
    dist.destroy_process_group()


def test_gloo_world_size_2(tmp_path):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_gloo_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()
