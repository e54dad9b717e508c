"""World-size-2 (and 3) gloo test of the N>1 path's host logic on CPU.

Each rank takes its slab from the native planner (vs_slab_plan, the same
code that lays out the device slabs), builds local [owned | ghost] vectors
and runs the inner PCGs with the fused kernel's schedule: z ghost planes
exchanged with the neighbouring ranks after every update (gloo send/recv),
ghost-plane d recomputed locally, partial sums combined in rank order.
The result must match the single-domain oracle (CPU restatement of the
reference) -- iteration count within 2 %, solution to 1e-10.
"""
import os
import socket

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def local_maps(sys_, plan, fams, velocity):
    """global index -> local index for the owned and ghost planes of a slab."""
    n = sys_.n
    g2l = {}
    for key, f in fams.items():
        lo, hi = plan["x_lo"], plan["x_hi"]
        if velocity:
            mask = sys_.masks[key]
            gids = sys_.face_ids(key)
        else:
            mask = sys_.fluid
            gids = np.full(mask.shape, -1, dtype=np.int64)
            gids[mask] = np.arange(sys_.m_p)
        def plane_ids(x):
            return gids[x % n][mask[x % n]]
        own = np.concatenate([plane_ids(x) for x in range(lo, hi)]) if hi > lo else np.zeros(0, int)
        assert own[0] == f["gstart"] if len(own) else True
        for k, gi in enumerate(own):
            g2l[int(gi)] = f["own_off"] + k
        for k, gi in enumerate(plane_ids(lo - 1)):
            g2l.setdefault(("lo", int(gi)), f["glo_off"] + k)
        for k, gi in enumerate(plane_ids(hi)):
            g2l.setdefault(("hi", int(gi)), f["ghi_off"] + k)
    return g2l


def _worker(rank, world, port, name, result_q):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        from oracle import voxoracle as vo
        from paper_2307_05266_b200.slabs import slab_plan

        g = load_golden(name)
        sys_ = vo.build_system(g["fluid"], int(g["flow_dir"]))
        plans = slab_plan(g["fluid"], world)
        me, lo_r, hi_r = plans[rank], (rank - 1) % world, (rank + 1) % world
        out = {}
        for op in ("A", "S"):
            velocity = op == "A"
            fams = {k: v for k, v in me["fam"].items() if (k != "p") == velocity}
            m_own = me["m_own"][0 if velocity else 1]
            m_all = me["m_all"][0 if velocity else 1]
            # global -> local; neighbours of owned DOFs resolve to owned or ghost slots
            nb_global = sys_.nb if velocity else None
            if velocity:
                owned_g = np.concatenate([sys_.axis_offsets[k] + np.arange(sys_.axis_counts[k])[
                    (np.argwhere(sys_.masks[k])[:, 0] >= me["x_lo"]) &
                    (np.argwhere(sys_.masks[k])[:, 0] < me["x_hi"])] for k in sorted(fams)])
                n_glob = sys_.m_u
            else:
                cells = np.argwhere(sys_.fluid)
                owned_g = np.arange(sys_.m_p)[(cells[:, 0] >= me["x_lo"]) & (cells[:, 0] < me["x_hi"])]
                n_glob = sys_.m_p
            g2l = local_maps(sys_, me, fams, velocity)
            own_local = np.array([g2l[int(gi)] for gi in owned_g])
            assert np.array_equal(own_local, np.arange(m_own))
            # local operator: dense restriction of the global operator to (owned, owned+ghost)
            inv_g = (1.0 / sys_.laplacian_diag) if velocity else \
                1.0 / vo.simple_inverse_diag(sys_)
            op_g = sys_.apply_laplacian if velocity else sys_.apply_simple
            cols = {}
            for j in range(n_glob):  # column probing (small golden systems only)
                e = np.zeros(n_glob)
                e[j] = 1.0
                colv = op_g(e)[owned_g]
                nz = np.nonzero(colv)[0]
                if len(nz):
                    cols[j] = (nz, colv[nz])
            # column j lives in local slot: owned, or the ghost plane that holds it
            def local_slot(j):
                if j in g2l:
                    return g2l[j]
                return g2l.get(("lo", j), g2l.get(("hi", j)))
            Aloc = np.zeros((m_own, m_all))
            for j, (rows, vals) in cols.items():
                sl = local_slot(j)
                assert sl is not None, "stencil reaches beyond the ghost planes"
                Aloc[rows, sl] += vals
            inv_l = inv_g[owned_g]

            def allsum(vals):
                t = torch.tensor(vals, dtype=torch.float64)
                parts = [torch.zeros_like(t) for _ in range(world)]
                dist.all_gather(parts, t)
                tot = parts[0].clone()
                for p_ in parts[1:]:
                    tot += p_
                return tot.numpy()

            def halo(vec):
                """fill ghost planes of vec (len m_all) from the neighbours' boundary planes."""
                reqs, bufs = [], {}
                for k, f in fams.items():
                    first = vec[f["own_off"]: f["own_off"] + f["first_cnt"]].copy()
                    last = vec[f["own_off"] + f["own"] - f["last_cnt"]: f["own_off"] + f["own"]].copy()
                    bufs[k] = (np.empty(f["glo_cnt"]), np.empty(f["ghi_cnt"]))
                    # first plane -> lower rank's ghost_hi, last plane -> upper rank's ghost_lo
                    reqs.append(dist.isend(torch.from_numpy(first), lo_r, tag=10 * (k if k != "p" else 3)))
                    reqs.append(dist.isend(torch.from_numpy(last), hi_r, tag=10 * (k if k != "p" else 3) + 1))
                for k, f in fams.items():
                    t_lo = torch.from_numpy(bufs[k][0])
                    t_hi = torch.from_numpy(bufs[k][1])
                    dist.recv(t_lo, lo_r, tag=10 * (k if k != "p" else 3) + 1)
                    dist.recv(t_hi, hi_r, tag=10 * (k if k != "p" else 3))
                    vec[f["glo_off"]: f["glo_off"] + f["glo_cnt"]] = t_lo.numpy()
                    vec[f["ghi_off"]: f["ghi_off"] + f["ghi_cnt"]] = t_hi.numpy()
                for r_ in reqs:
                    r_.wait()

            rng = np.random.default_rng(7)
            rhs_g = rng.standard_normal(n_glob)
            proj = not velocity
            m_glob = n_glob
            rhs = rhs_g[owned_g].copy()
            if proj:
                rhs = rhs - allsum([rhs.sum()])[0] / m_glob
            # fused-kernel schedule: r = -rhs, z = M r, z halo; P1 d (+ghost d); P2 ...
            x = np.zeros(m_own)
            r = 0.0 - rhs
            z = np.zeros(m_all)
            z[:m_own] = r * inv_l
            halo(z)
            s5 = allsum([r @ z[:m_own], z[:m_own] @ z[:m_own], r @ r, z[:m_own].sum(), r.sum()])
            mu = s5[3] / m_glob if proj else 0.0
            rz = s5[0] - mu * s5[4] if proj else s5[0]
            zz = s5[1] - mu * s5[3] if proj else s5[1]
            ref = np.sqrt(zz)
            dold = np.zeros(m_all)
            its, beta = 0, 0.0
            for k_ in range(5000):
                zc = z - mu if proj else z
                d = zc if k_ == 0 else zc + beta * dold   # owned + ghost planes alike
                q = Aloc @ d
                dq = allsum([d[:m_own] @ q])[0]
                alpha = rz / dq
                x -= alpha * d[:m_own]
                r -= alpha * q
                z = np.zeros(m_all)
                z[:m_own] = r * inv_l
                halo(z)
                s5 = allsum([r @ z[:m_own], z[:m_own] @ z[:m_own], r @ r, z[:m_own].sum(), r.sum()])
                if proj:
                    mu = s5[3] / m_glob
                    rz_new, zz = s5[0] - mu * s5[4], s5[1] - mu * s5[3]
                else:
                    rz_new, zz = s5[0], s5[1]
                beta, rz = rz_new / rz, rz_new
                its = k_ + 1
                dold = d
                if np.sqrt(zz) / ref < 1e-12:
                    break
            xs = [torch.zeros(0)] * world
            xg = torch.from_numpy(np.concatenate([owned_g.astype(float), x]))
            sizes = [torch.zeros(1) for _ in range(world)]
            dist.all_gather(sizes, torch.tensor([float(len(x))]))
            mx = int(max(s_.item() for s_ in sizes))
            pad = torch.zeros(2 * mx, dtype=torch.float64)
            pad[: 2 * len(x)] = xg
            allx = [torch.zeros(2 * mx, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(allx, pad)
            full = np.zeros(n_glob)
            for s_, t in zip(sizes, allx):
                cnt = int(s_.item())
                idx = t[:cnt].numpy().astype(int)
                full[idx] = t[cnt: 2 * cnt].numpy()
            out[op] = (its, full, rhs_g)
        if rank == 0:
            result_q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["pack2d", "rand3d"])
def test_distributed_slab_pcg_matches_oracle(name, world):
    import multiprocessing as mp

    from oracle import voxoracle as vo

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = load_golden(name)
    sys_ = vo.build_system(g["fluid"], int(g["flow_dir"]))
    its, x, rhs = res["A"]
    xo, io = vo.solve_velocity(sys_, rhs, 1e-12)
    assert abs(its - io) <= max(1, int(0.02 * io))
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    its, z, rhs = res["S"]
    zo, io = vo.solve_simple(sys_, rhs, 1e-12)
    assert abs(its - io) <= max(1, int(0.02 * io))
    assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo)


def test_slab_plan_consistency():
    """ghost planes of slab s are the neighbours' boundary planes, sizes match."""
    from paper_2307_05266_b200.slabs import slab_plan

    g = load_golden("spheres3d")
    for R in (2, 3, 5):
        plans = slab_plan(g["fluid"], R)
        for s, me in enumerate(plans):
            lo, hi = plans[(s - 1) % R], plans[(s + 1) % R]
            for key, f in me["fam"].items():
                assert f["glo_cnt"] == lo["fam"][key]["last_cnt"]
                assert f["ghi_cnt"] == hi["fam"][key]["first_cnt"]
            assert me["m_all"][0] >= me["m_own"][0] and me["m_all"][1] >= me["m_own"][1]
        assert sum(p["m_own"][1] for p in plans) == int(g["fluid"].sum())
        assert sum(p["m_own"][0] for p in plans) == int(g["m_u"])
