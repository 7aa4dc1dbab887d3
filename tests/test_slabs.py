"""z-slab decomposition: host tables (CPU, incl. a world_size-2 gloo run) and the single-GPU
lockstep emulation of 2-4 slabs against the one-slab operator."""
import os
import socket

import numpy as np
import pytest

from paper_2205_08909_b200 import dofs, mesh as pmesh, slabs
from _problems import gpu_operator, hist_array, host_tables, rel, seeded_rhs


def _global(cells, p):
    m = pmesh.build_cartesian_mesh(cells)
    return m, dofs.distribute_dofs(m, p, 1, constrain_boundary=True)


def _global_lattice_of(h, p):
    node, I, J, K = slabs._lattice_ids(h, 0)
    nx, ny, nz = h.cells_per_dim
    out = np.empty(h.n_dofs, dtype=np.int64)
    out[node] = I + (nx * p + 1) * (J + (ny * p + 1) * K)
    return out


@pytest.mark.parametrize("cells,p,G", [((3, 2, 5), 2, 2), ((4, 3, 7), 3, 3), ((2, 2, 8), 5, 4)])
def test_slab_tables_against_global_numbering(cells, p, G):
    m, h = _global(cells, p)
    lat_of_global = _global_lattice_of(h, p)           # global node -> lattice id
    glob_of_lat = np.empty_like(lat_of_global)
    glob_of_lat[lat_of_global] = np.arange(h.n_dofs)   # lattice id -> global node (reference numbering)
    layers = slabs.slab_layers(cells[2], G)
    assert sum(n for _, n in layers) == cells[2] and layers[0][0] == 0
    sl = [slabs.build_slab(m, p, z0, n) for z0, n in layers]
    covered = np.zeros(h.n_dofs, dtype=int)
    for g, s in enumerate(sl):
        gl = glob_of_lat[s.global_nodes]                # local node -> global node id
        # numbering: the slab's block table maps onto the reference's global one, cell by cell
        nxy = cells[0] * cells[1]
        loc = dofs.expand_batch(s.handler, np.arange(s.handler.n_cells))
        ref = dofs.expand_batch(h, np.arange(s.handler.n_cells) + s.z0 * nxy)
        assert np.array_equal(gl[loc], ref)
        # Dirichlet set = global set restricted to the slab
        assert np.array_equal(np.sort(gl[s.handler.constrained_dofs]),
                              np.intersect1d(h.constrained_dofs, gl))
        covered[gl] += 1
        # ghost map: shared plane = intersection of the two slabs' DoFs
        if g + 1 < G:
            up = sl[g + 1]
            mine = gl[slabs.interface_plane_nodes(s, "upper")]
            theirs = glob_of_lat[up.global_nodes][slabs.interface_plane_nodes(up, "lower")]
            cells_lo = np.arange(s.handler.n_cells) + s.z0 * nxy
            cells_up = np.arange(up.handler.n_cells) + up.z0 * nxy
            shared = np.intersect1d(np.unique(dofs.expand_batch(h, cells_lo)),
                                    np.unique(dofs.expand_batch(h, cells_up)))
            assert np.array_equal(np.sort(mine), shared) and np.array_equal(mine, theirs)
    assert covered.min() == 1 and covered.max() == 2 and (covered == 2).sum() == (G - 1) * (
        (cells[0] * p + 1) * (cells[1] * p + 1))


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cells, p = (3, 2, 6), 3
    m = pmesh.build_cartesian_mesh(cells)
    z0, n = slabs.slab_layers(cells[2], world)[rank]
    s = slabs.build_slab(m, p, z0, n)
    ok = True
    # neighbours agree on the ghost map (global lattice ids of the shared plane, same order)
    if s.has_upper:
        mine = torch.from_numpy(s.global_nodes[slabs.interface_plane_nodes(s, "upper")])
        dist.send(mine, rank + 1)
    if s.has_lower:
        mine = torch.from_numpy(s.global_nodes[slabs.interface_plane_nodes(s, "lower")])
        theirs = torch.empty_like(mine)
        dist.recv(theirs, rank - 1)
        ok = ok and bool(torch.equal(mine, theirs))
    # owned-DoF count and a seven-scalar all-reduce, the collective of one merged iteration
    owned = s.handler.n_dofs - (len(interface := slabs.interface_plane_nodes(s, "lower")) if s.has_lower else 0)
    t = torch.tensor([float(owned)] + [float(rank + 1)] * 6, dtype=torch.float64)
    dist.all_reduce(t)
    total = int(np.prod([c * p + 1 for c in cells]))
    ok = ok and int(t[0]) == total and float(t[1]) == world * (world + 1) / 2
    q.put((rank, ok))
    dist.destroy_process_group()


def test_slab_host_logic_world_size_2_gloo():
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = sorted(q.get(timeout=120) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert results == [(0, True), (1, True)]


@pytest.mark.parametrize("cells,p,G", [((4, 3, 8), 3, 2), ((3, 3, 9), 2, 3), ((2, 2, 8), 5, 4)])
def test_slab_renumbering_with_remote_category(cells, p, G):
    """Per-slab `renumber_optimized` with the interface planes in the remote-shared category (the reference's
    empty placeholder, dofs.py:307-310): bijection, category order single-batch < multi-batch < remote <
    constrained, the planes contiguous, and -- the oracle of SURVEY.md 8e -- the same relative order as the
    plain renumbering inside every category."""
    m, _ = _global(cells, p)
    for z0, n in slabs.slab_layers(cells[2], G):
        s = slabs.build_slab(m, p, z0, n)
        plan = dofs.make_batches(s.mesh, dofs.batch_size(p, 1, 8), "morton")
        r = slabs.renumber_slab(s, plan)
        h, hr = s.handler, r.handler
        perm = hr.permutation
        assert np.array_equal(np.sort(perm), np.arange(h.n_dofs))
        assert np.array_equal(np.sort(r.global_nodes), np.sort(s.global_nodes))
        assert np.array_equal(r.global_nodes[perm], s.global_nodes)
        # expansions follow the permutation (reference tests/test_dofs.py:214-221)
        cells_all = np.arange(h.n_cells)
        assert np.array_equal(dofs.expand_batch(hr, cells_all), perm[dofs.expand_batch(h, cells_all)])
        # constrained tail, remote block right before it, contiguous
        k = len(h.constrained_dofs)
        assert np.array_equal(hr.constrained_dofs, np.arange(h.n_dofs - k, h.n_dofs))
        planes = [slabs.interface_plane_nodes(s, side) for side, has in (("lower", s.has_lower), ("upper", s.has_upper)) if has]
        remote = np.concatenate(planes) if planes else np.empty(0, dtype=np.int64)
        con = np.zeros(h.n_dofs, bool)
        con[h.constrained_dofs] = True
        free_remote = remote[~con[remote]]
        new_remote = np.sort(perm[free_remote])
        assert np.array_equal(new_remote, np.arange(h.n_dofs - k - len(free_remote), h.n_dofs - k))
        # same relative order as the plain renumbering among the unknowns that are neither remote nor constrained
        plain = dofs.renumber_optimized(h, plan).permutation
        rest = np.setdiff1d(np.arange(h.n_dofs), np.concatenate([free_remote, h.constrained_dofs]))
        assert np.array_equal(np.argsort(plain[rest]), np.argsort(perm[rest]))


@pytest.mark.gpu
@pytest.mark.parametrize("cells,p,G,deform,bz", [((5, 4, 9), 5, 2, 0.0, 0), ((6, 5, 12), 3, 3, 0.0, 0),
                                                 ((4, 4, 17), 5, 4, 0.0, 0), ((4, 3, 6), 3, 2, 0.1, 0),
                                                 # bricks one cell layer deep: slabs of 4-5 brick layers, so the
                                                 # interface layers go out first (middle slabs: one wrap-around launch)
                                                 ((5, 4, 13), 5, 3, 0.0, 1), ((4, 3, 9), 3, 2, 0.1, 1)])
def test_slab_group_equals_single_slab_on_one_gpu(cells, p, G, deform, bz):
    """G slabs stepped in lockstep on one GPU (device-to-device plane copies stand in for NCCL)
    against the one-slab operator: apply and diagonal at 1e-12, merged-CG history at 1e-10."""
    from paper_2205_08909_b200 import solvers as S
    from paper_2205_08909_b200.operator import MatrixFreeOperator, OperatorSpec
    variant = "final_tensor_load" if deform else "affine"
    m, h, plan = host_tables(cells, p, deform=deform)
    op1 = gpu_operator(m, h, plan, p, p + 1, variant=variant)
    lat = _global_lattice_of(h, p)
    glob_of_lat = np.empty_like(lat)
    glob_of_lat[lat] = np.arange(h.n_dofs)
    sl = [slabs.build_slab(m, p, z0, n) for z0, n in slabs.slab_layers(cells[2], G)]
    if G == 3:  # one case with per-slab optimized numbering (interface planes in the remote-shared category)
        sl = [slabs.renumber_slab(s, dofs.make_batches(s.mesh, dofs.batch_size(p, 1, 8), "morton")) for s in sl]
    ops = []
    for s in sl:
        plan_s = dofs.make_batches(s.mesh, dofs.batch_size(p, 1, 8), "morton")
        ops.append(MatrixFreeOperator(OperatorSpec("laplace", 1, p, p + 1, pmesh.GeometryVariant(variant)),
                                      s.mesh, s.handler, plan_s, slab_z0=s.z0,
                                      global_cells_z=s.global_cells_z, brick=(0, 0, bz)))
    if bz:
        assert all(o.info()["brick"][2] == bz and o.info()["n_bricks"] >= 3 for o in ops)
    maps = [glob_of_lat[s.global_nodes] for s in sl]
    group = slabs.SlabGroup(ops)
    u = np.random.default_rng(3).standard_normal(h.n_dofs)
    ref = op1.apply(u)
    for gl, out in zip(maps, group.apply([u[gl] for gl in maps])):
        assert rel(out, ref[gl]) < 1e-12
    dref = op1.compute_diagonal().inverse_diagonal
    for gl, d in zip(maps, group.compute_diagonal()):
        assert rel(d, dref[gl]) < 1e-12
    b = seeded_rhs(h)
    cfg = S.SolverConfig(fixed_iterations=40)
    one = S.solve("combined_pcg", op1, b, minv=op1.compute_diagonal(), config=cfg)
    many = group.solve("combined_pcg", [b[gl] for gl in maps], cfg)
    H1 = hist_array(one.history)
    for gl, r in zip(maps, many):
        assert r.iterations == 40
        assert rel(hist_array(r.history)[:30], H1[:30]) < 1e-10
        assert rel(r.x, one.x[gl]) < 1e-9
    # caller-supplied preconditioner per slab (the single-slab diagonal restricted to the slab)
    custom = group.solve("combined_pcg", [b[gl] for gl in maps], cfg, minvs=[dref[gl] for gl in maps])
    for gl, r in zip(maps, custom):
        assert rel(hist_array(r.history)[:30], H1[:30]) < 1e-10
    # standard (unfused) PCG and CG on the slabs (BASELINE configs[3]/[4] "standard vs merged" arm)
    for variant in ("pcg", "cg"):
        one_s = S.solve(variant, op1, b, minv=op1.compute_diagonal() if variant == "pcg" else None, config=cfg)
        many_s = group.solve(variant, [b[gl] for gl in maps], cfg)
        Hs = hist_array(one_s.history)
        for gl, r in zip(maps, many_s):
            assert r.iterations == 40 and r.matvecs == 40
            assert rel(hist_array(r.history)[:30], Hs[:30]) < 1e-10, variant
            assert rel(r.x, one_s.x[gl]) < 1e-9, variant
    # tolerance-terminated run agrees on the iteration count
    one = S.solve("combined_pcg", op1, b, minv=op1.compute_diagonal(), config=S.SolverConfig(tolerance=1e-7))
    many = group.solve("combined_pcg", [b[gl] for gl in maps], S.SolverConfig(tolerance=1e-7))
    assert all(abs(r.iterations - one.iterations) <= 1 and r.converged for r in many)


def test_three_component_slab_tables():
    """build_slab with 3 components: interleaved unknowns, whole-node constraints, per-node lattice map."""
    m = pmesh.build_cartesian_mesh((3, 2, 6))
    s1 = slabs.build_slab(m, 2, 2, 2)
    s3 = slabs.build_slab(m, 2, 2, 2, components=3)
    assert s3.handler.components == 3 and s3.handler.n_dofs == 3 * s1.handler.n_dofs
    assert np.array_equal(s3.global_nodes, s1.global_nodes)
    c1 = s1.handler.constrained_dofs
    assert np.array_equal(s3.handler.constrained_dofs, (3 * c1[:, None] + np.arange(3)).ravel())
    ref = dofs.distribute_dofs(s1.mesh, 2, 3, constrain_boundary=False)
    assert np.array_equal(s3.handler.cell_index_blocks, ref.cell_index_blocks)


@pytest.mark.gpu
@pytest.mark.parametrize("cells,p,G,deform", [((5, 4, 9), 5, 2, 0.0), ((4, 3, 8), 3, 3, 0.1)])
def test_three_component_slab_group_equals_single_slab(cells, p, G, deform):
    """BP4-type operator (3 components) on G slabs in lockstep against the one-slab operator: apply, merged PCG
    and standard PCG; the interface planes of all three component fields travel in one buffer."""
    from paper_2205_08909_b200 import solvers as S
    from paper_2205_08909_b200.operator import MatrixFreeOperator, OperatorSpec
    variant = "final_tensor_load" if deform else "affine"
    m, h, plan = host_tables(cells, p, deform=deform, components=3)
    op1 = gpu_operator(m, h, plan, p, p + 1, variant=variant)
    hs = dofs.distribute_dofs(m, p, 1, constrain_boundary=True)
    lat = _global_lattice_of(hs, p)
    glob_of_lat = np.empty_like(lat)
    glob_of_lat[lat] = np.arange(hs.n_dofs)
    sl = [slabs.build_slab(m, p, z0, n, components=3) for z0, n in slabs.slab_layers(cells[2], G)]
    ops = []
    for s in sl:
        plan_s = dofs.make_batches(s.mesh, dofs.batch_size(p, 3, 8), "morton")
        ops.append(MatrixFreeOperator(OperatorSpec("laplace", 3, p, p + 1, pmesh.GeometryVariant(variant)),
                                      s.mesh, s.handler, plan_s, slab_z0=s.z0, global_cells_z=s.global_cells_z))
    node_maps = [glob_of_lat[s.global_nodes] for s in sl]
    maps = [(3 * nm[:, None] + np.arange(3)[None, :]).ravel() for nm in node_maps]
    group = slabs.SlabGroup(ops)
    rng = np.random.default_rng(4)
    u = rng.standard_normal(h.n_dofs)
    ref = op1.apply(u)
    for gl, out in zip(maps, group.apply([u[gl] for gl in maps])):
        assert rel(out, ref[gl]) < 1e-12
    dref = op1.compute_diagonal().inverse_diagonal          # one value per node
    for nm, d in zip(node_maps, group.compute_diagonal()):
        assert d.shape == nm.shape and rel(d, dref[nm]) < 1e-12
    b = rng.uniform(-1, 1, h.n_dofs)
    b[h.constrained_dofs] = 0.0
    cfg = S.SolverConfig(fixed_iterations=30)
    for name in ("combined_pcg", "pcg", "combined_cg"):
        mv = op1.compute_diagonal() if name != "combined_cg" else None
        one = S.solve(name, op1, b, minv=mv, config=cfg)
        many = group.solve(name, [b[gl] for gl in maps], cfg)
        H1 = hist_array(one.history)
        for gl, r in zip(maps, many):
            assert r.iterations == 30
            assert rel(hist_array(r.history)[:25], H1[:25]) < 1e-10, name
            assert rel(r.x, one.x[gl]) < 1e-9, name
    custom = group.solve("combined_pcg", [b[gl] for gl in maps], cfg, minvs=[dref[nm] for nm in node_maps])
    one = S.solve("combined_pcg", op1, b, minv=op1.compute_diagonal(), config=cfg)
    for gl, r in zip(maps, custom):
        assert rel(hist_array(r.history)[:25], hist_array(one.history)[:25]) < 1e-10


@pytest.mark.gpu
def test_nccl_binding_single_rank():
    """The run-time NCCL binding (dlopen of the libnccl torch ships): unique id, communicator with
    one rank, and the seven-sum all-reduce inside a one-slab group solve."""
    import torch  # noqa: F401  (loads libnccl.so.2 into the process)
    from paper_2205_08909_b200 import solvers as S
    uid = slabs.new_unique_id()
    assert len(uid) == 128 and any(uid)
    slabs.init_comm(0, uid, 0, 1)
    m, h, plan = host_tables((5, 4, 6), 3)
    op = gpu_operator(m, h, plan, 3, 4)
    b = seeded_rhs(h)
    cfg = S.SolverConfig(fixed_iterations=25)
    one = S.solve("combined_pcg", op, b, minv=op.compute_diagonal(), config=cfg)
    grp = slabs.SlabGroup([op]).solve("combined_pcg", [b], cfg)[0]
    assert rel(hist_array(grp.history), hist_array(one.history)) < 1e-12
    assert rel(grp.x, one.x) < 1e-12


@pytest.mark.gpu
def test_nccl_send_recv_to_self_through_group_exchange(monkeypatch):
    """ncclSend / ncclRecv, their dtype constant and the stream ordering of `group_exchange`, on one GPU: a
    middle slab (neighbours below and above) on a one-rank communicator with both peers redirected to the
    rank itself (MFCG_NCCL_SELF_PEER=1; send-to-self inside one NCCL group is legal).  Sends and receives to
    the same peer match in posting order, so the slab receives its own bottom / top plane contributions and
    adds them once more: v doubles on the two interface planes and is untouched elsewhere, compared with the
    same slab as a stand-alone operator (no neighbours, same constraint set)."""
    import torch  # noqa: F401  (loads libnccl.so.2 into the process)
    from paper_2205_08909_b200.operator import MatrixFreeOperator, OperatorSpec
    monkeypatch.setenv("MFCG_NCCL_SELF_PEER", "1")
    slabs.init_comm(0, slabs.new_unique_id(), 0, 1)
    p, cells = 3, (5, 4, 12)
    gm = pmesh.build_cartesian_mesh(cells)
    s = slabs.build_slab(gm, p, 4, 4)           # cell layers 4..7 of 12: neighbours on both sides
    assert s.has_lower and s.has_upper
    plan = dofs.make_batches(s.mesh, dofs.batch_size(p, 1, 8), "morton")
    spec = OperatorSpec("laplace", 1, p, p + 1, pmesh.GeometryVariant.AFFINE)
    op_mid = MatrixFreeOperator(spec, s.mesh, s.handler, plan, slab_z0=s.z0, global_cells_z=s.global_cells_z)
    # the same cells as a mesh of their own: extents scaled so that h is the same, same constraint set
    alone_mesh = pmesh.build_cartesian_mesh(s.mesh.cells_per_dim, (1.0, 1.0, 4.0 / 12.0))
    op_alone = MatrixFreeOperator(spec, alone_mesh, s.handler, plan)
    u = np.random.default_rng(5).standard_normal(s.handler.n_dofs)
    got = slabs.SlabGroup([op_mid]).apply([u])[0]
    ref = op_alone.apply(u)
    lower, upper = slabs.interface_plane_nodes(s, "lower"), slabs.interface_plane_nodes(s, "upper")
    con = np.zeros(s.handler.n_dofs, bool)
    con[s.handler.constrained_dofs] = True
    expect = ref.copy()
    for plane in (lower, upper):
        free = plane[~con[plane]]
        expect[free] = 2.0 * ref[free]          # own contribution received once more from "the neighbour"
    assert rel(got, expect) < 1e-12
