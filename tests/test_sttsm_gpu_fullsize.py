"""Parity at BASELINE.json's full sizes.

The numpy oracle is too slow for whole full-size problems, so these tests use
(1) the oracle on sampled top-level subtrees of the full problem,
(2) exact structural identities (a permutation / truncation X turns the
    change of basis into a pure re-indexing of A: bitwise equality),
(3) a multilinear checksum  C(v,..,v) == A(X^T v,..,X^T v)  evaluated
    independently in torch fp64, and
(4) linearity in A.
"""

import itertools
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_1301_7744_b200 as bs  # noqa: E402
from oracle import bcss_oracle as orc  # noqa: E402
from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device  # noqa: E402

CFG = {2: (3, 512, 512, 32, 32), 3: (4, 192, 192, 16, 16), 4: (5, 96, 96, 8, 8), 5: (4, 512, 256, 32, 32)}


def run(cfg, a, x):
    m, n, p, ba, bc = cfg
    plan = bs.SttsmPlan(m, n, p, ba, bc)
    c = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.run(a, x, c)
    torch.cuda.synchronize()
    plan.close()
    return c


@pytest.mark.parametrize("cfg_id,units", [(2, [0, 1, 15]), (3, [0, 1]), (3, [11]), (4, [0, 1]), (4, [11]),
                                          (5, [0])])
def test_full_size_subtrees_match_oracle(cfg_id, units):
    """Oracle on whole top-level subtrees of the full-size problem: the
    cheapest ones, and the largest subtree (unit 11) of configs 3 and 4, whose
    parents reach every tile height of the b_A = 8 / 16 shapes; config 5's
    unit 0 is 7.1 % of the headline workload's flops (about 25 s of CPU)."""
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 11 + cfg_id)
    x = random_matrix_device(p, n, 12 + cfg_id)
    c = run(CFG[cfg_id], a, x).cpu().numpy()
    want = orc.sttsm_bcss_packed(a.cpu().numpy(), x.cpu().numpy(), m, n, ba, bc, units=units)
    mask = np.zeros(bs.simplex_count(p // bc, m), dtype=bool)
    for r in bs.SttsmPlan(m, n, p, ba, bc, units=units).c_block_ranks():
        mask[r] = True
    got_b = c.reshape(-1, bc**m)[mask]
    want_b = want.reshape(-1, bc**m)[mask]
    assert orc.rel_frobenius(got_b, want_b) <= 1e-12
    assert orc.max_rel(got_b, want_b) <= 1e-10


def _block_perm(nbar, b, seed):
    """X = permutation matrix mapping output index j -> input index pi(j) with
    pi = (block permutation sigma) x (within-block permutation tau)."""
    rng = np.random.default_rng(seed)
    sigma = rng.permutation(nbar)
    tau = rng.permutation(b)
    return sigma, tau


@pytest.mark.parametrize("cfg_id", [2, 3, 4, 5])
def test_permutation_x_reindexes_a_bitwise(cfg_id):
    """X[j, pi(j)] = 1: C[j_0..j_{m-1}] = A[pi(j_0)..pi(j_{m-1})] exactly (every
    output is one product of ones with one entry of A).  With p < n (config 5)
    X is a truncated permutation.  Checks every C block at full size."""
    m, n, p, ba, bc = CFG[cfg_id]
    assert ba == bc
    nbar, pbar = n // ba, p // bc
    sigma, tau = _block_perm(nbar, ba, 100 + cfg_id)
    sigma = sigma[:pbar]
    pi = (sigma[:, None] * ba + tau[None, :]).reshape(-1)  # output row j -> input col
    x = torch.zeros(p, n, dtype=torch.float64, device="cuda")
    x[torch.arange(p, device="cuda"), torch.as_tensor(pi, device="cuda")] = 1.0
    a = random_bcss_device(m, n, ba, 21 + cfg_id)
    c = run(CFG[cfg_id], a, x)
    blocks_a = a.view(-1, *([ba] * m))  # torch axes = F-order modes reversed
    blocks_c = c.view(-1, *([bc] * m))
    tau_t = torch.as_tensor(tau, device="cuda")
    keys = list(itertools.combinations_with_replacement(range(pbar), m))
    # group output blocks by the canonicalize permutation of their source index
    for r, key in enumerate(keys):
        src = tuple(int(sigma[j]) for j in key)
        canon, mapping = bs.canonicalize(src)
        blk = blocks_a[bs.hypertriangle_rank(canon, nbar)]
        # logical block (modes d) = stored block transposed by mapping; torch axes reversed
        order = [m - 1 - mapping[m - 1 - ax] for ax in range(m)]
        logical = blk.permute(*order)
        for ax in range(m):
            logical = logical.index_select(ax, tau_t)
        assert torch.equal(blocks_c[r], logical), (key, src)


def _mult(key):
    cnt = {}
    for v in key:
        cnt[v] = cnt.get(v, 0) + 1
    out = math.factorial(len(key))
    for c in cnt.values():
        out //= math.factorial(c)
    return out


def multilinear_form(packed, m, dim, b, v):
    """sum over the dense tensor of T[i] * prod_d v[i_d], from canonical blocks
    with their orbit multiplicities (each block's entries summed densely)."""
    g = dim // b
    keys = list(itertools.combinations_with_replacement(range(g), m))
    blocks = packed.view(len(keys), *([b] * m))
    vb = v.view(g, b)
    idx = torch.as_tensor(keys, device=v.device)           # (nblk, m)
    mult = torch.as_tensor([_mult(k) for k in keys], dtype=torch.float64, device=v.device)
    vals, absvals = torch.zeros((), dtype=torch.float64, device=v.device), 0.0
    step = 256
    letters = "abcdefgh"[:m]
    for s in range(0, len(keys), step):
        blk = blocks[s:s + step]
        ops = [vb[idx[s:s + step, m - 1 - ax]] for ax in range(m)]  # torch axis ax = mode m-1-ax
        expr = "z" + letters + "," + ",".join("z" + letters[ax] for ax in range(m)) + "->z"
        per = torch.einsum(expr, blk, *ops)
        vals = vals + (mult[s:s + step] * per).sum()
        per_abs = torch.einsum(expr, blk.abs(), *[o.abs() for o in ops])
        absvals += float((mult[s:s + step] * per_abs).sum())
    return float(vals), absvals


@pytest.mark.parametrize("cfg_id", [2, 3, 4, 5])
def test_multilinear_checksum(cfg_id):
    """C(v, .., v) == A(X^T v, .., X^T v) for a random v (torch fp64)."""
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 31 + cfg_id)
    x = random_matrix_device(p, n, 32 + cfg_id)
    c = run(CFG[cfg_id], a, x)
    v = torch.randn(p, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
    lhs, lhs_abs = multilinear_form(c, m, p, bc, v)
    rhs, rhs_abs = multilinear_form(a, m, n, ba, x.t() @ v)
    assert abs(lhs - rhs) <= 1e-11 * max(lhs_abs, rhs_abs)


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_linearity_in_a(cfg_id):
    m, n, p, ba, bc = CFG[cfg_id]
    a1 = random_bcss_device(m, n, ba, 41)
    a2 = random_bcss_device(m, n, ba, 42)
    x = random_matrix_device(p, n, 43)
    c1, c2 = run(CFG[cfg_id], a1, x), run(CFG[cfg_id], a2, x)
    c12 = run(CFG[cfg_id], a1 - 0.5 * a2, x)
    ref = c1 - 0.5 * c2
    assert float((c12 - ref).norm() / ref.norm()) <= 1e-13


@pytest.mark.parametrize("cfg_id,waves", [(2, 4), (3, 3), (4, 2)])
def test_pipelined_host_run(cfg_id, waves):
    """run_host with the transfer/compute pipeline (pinned buffers, chunk-gated
    top level, mirrored C order, one D2H per wave) returns exactly what the same
    plan computes on device buffers, and matches the plain plan to 1e-13 (the
    mirrored plan contracts the C modes in the opposite order)."""
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 51 + cfg_id)
    x = random_matrix_device(p, n, 52 + cfg_id)
    plain = run(CFG[cfg_id], a, x).cpu()
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=waves)
    assert 2 <= plan.stats()["waves"] <= waves
    c_dev = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64, device="cuda")
    plan.run(a, x, c_dev)
    torch.cuda.synchronize()
    want = c_dev.cpu()
    assert float((want - plain).norm() / plain.norm()) <= 1e-13
    a_h, x_h = a.cpu().pin_memory(), x.cpu().pin_memory()
    c_h = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(a_h.numpy(), x_h.numpy(), c_h.numpy())
    assert torch.equal(c_h, want)
    c_h.fill_(float("nan"))
    plan.run_host(a_h.numpy(), x_h.numpy(), c_h.numpy())  # reuse of streams / events
    assert torch.equal(c_h, want)


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_mirrored_plan_matches_oracle_subtree(cfg_id):
    """The mirrored C order against the numpy oracle on a reduced problem of the
    same block sizes (p̄ = 4 row blocks, all C blocks)."""
    m, n, p, ba, bc = CFG[cfg_id]
    n, p = 4 * ba, 4 * bc
    a = random_bcss_device(m, n, ba, 71 + cfg_id)
    x = random_matrix_device(p, n, 72 + cfg_id)
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=3)
    c = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.run(a, x, c)
    torch.cuda.synchronize()
    want = orc.sttsm_bcss_packed(a.cpu().numpy(), x.cpu().numpy(), m, n, ba, bc)
    got = c.cpu().numpy()
    assert orc.rel_frobenius(got, want) <= 1e-12


@pytest.mark.parametrize("cfg_id,world", [(2, 4), (3, 4), (4, 8), (5, 8)])
def test_s5_partial_plans_reassemble_c_bitwise(cfg_id, world):
    """The S5 multi-GPU schedule on one GPU: every virtual rank's owner plan
    (levels m-1..m-2, stop-level output) and subtree plan (start calls from the
    exchanged T(m-2) slices) run in turn; the union of their C blocks equals
    the single-plan result bit for bit."""
    from paper_1301_7744_b200.distributed import s5_schedule
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 61 + cfg_id)
    x = random_matrix_device(p, n, 62 + cfg_id)
    want = run(CFG[cfg_id], a, x)
    owners, subs = s5_schedule(m, n, p, ba, bc, world)
    slices = {}
    for r in range(world):
        if not owners[r]:
            continue
        pl = bs.SttsmPlan(m, n, p, ba, bc, units=owners[r], stop_level=m - 2)
        t2 = torch.empty(pl.c_elems, dtype=torch.float64, device="cuda")
        pl.run(a, x, t2)
        calls = pl.level_calls(m - 2)
        size = t2.numel() // len(calls)
        for i, c in enumerate(calls):
            slices[c] = t2[i * size:(i + 1) * size]
        pl.close()
    c = torch.full_like(want, float("nan"))
    for r in range(world):
        if not subs[r]:
            continue
        inp = torch.cat([slices[cl] for cl in subs[r]])
        pl = bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 2, start_calls=subs[r])
        part = torch.full_like(want, float("nan"))
        pl.run(inp, x, part)
        idx = torch.as_tensor(pl.c_block_ranks(), device="cuda")
        c.view(-1, bc**m)[idx] = part.view(-1, bc**m)[idx]
        pl.close()
    torch.cuda.synchronize()
    assert torch.equal(c, want)


@pytest.mark.parametrize("cfg_id,world,force", [(5, 8, False), (3, 8, True), (4, 8, True)])
def test_s5_helper_tasks_reassemble_c_bitwise(cfg_id, world, force):
    """The S5 schedule with helpers on one GPU: an owner computes T(m-1)[u]
    (top-level plan) and the level-(m-2) children it keeps (start plan with a
    child subset); its helper computes the handed-over children from a copy of
    T(m-1)[u]; every release group's subtree plan finishes the C blocks.  The
    union equals the single-plan C bit for bit."""
    from paper_1301_7744_b200.distributed import s5_tasks
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 81 + cfg_id)
    x = random_matrix_device(p, n, 82 + cfg_id)
    want = run(CFG[cfg_id], a, x)
    sc = s5_tasks(m, n, p, ba, bc, world, force_helper=force)
    assert sc["helper"], "the schedule should hand work to a helper"
    slices, tops = {}, {}

    def produce(pl, inp):
        out = torch.empty(pl.c_elems, dtype=torch.float64, device="cuda")
        pl.run(inp, x, out)
        calls = pl.level_calls(m - 2)
        size = out.numel() // len(calls)
        for i, c in enumerate(calls):
            assert c not in slices
            slices[c] = out[i * size:(i + 1) * size]
        pl.close()

    for r in range(world):
        for u in sc["owners"][r]:
            if u in sc["helper"]:
                pt = bs.SttsmPlan(m, n, p, ba, bc, units=[u], stop_level=m - 1)
                tops[u] = torch.empty(pt.c_elems, dtype=torch.float64, device="cuda")
                pt.run(a, x, tops[u])
                pt.close()
                produce(bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 1, start_calls=[(u,)],
                                     start_children=sc["own_children"][u], stop_level=m - 2), tops[u])
        mine = [u for u in sc["owners"][r] if u not in sc["helper"]]
        if mine:
            produce(bs.SttsmPlan(m, n, p, ba, bc, units=mine, stop_level=m - 2), a)
    for u, (h, kids) in sc["helper"].items():
        produce(bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 1, start_calls=[(u,)], start_children=kids,
                             stop_level=m - 2), tops[u].clone())
    assert len(slices) == sum(u + 1 for u in range(p // bc))
    c = torch.full_like(want, float("nan"))
    for r in range(world):
        for lo, hi, _ in sc["groups"][r]:
            calls = sc["subs"][r][lo:hi]
            pl = bs.SttsmPlan(m, n, p, ba, bc, start_level=m - 2, start_calls=calls)
            part = torch.full_like(want, float("nan"))
            pl.run(torch.cat([slices[cl] for cl in calls]), x, part)
            idx = torch.as_tensor(pl.c_block_ranks(), device="cuda")
            c.view(-1, bc**m)[idx] = part.view(-1, bc**m)[idx]
            pl.close()
    torch.cuda.synchronize()
    assert torch.equal(c, want)


@pytest.mark.parametrize("cfg_id", [3, 4])
def test_unit_subsets_and_workspace_waves_are_bitwise_identical(cfg_id):
    """Plans restricted to unit subsets write exactly their C blocks (others
    untouched), and a workspace limit that forces several waves changes
    nothing: every variant reproduces the single-plan C bit for bit."""
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 71 + cfg_id)
    x = random_matrix_device(p, n, 72 + cfg_id)
    want = run(CFG[cfg_id], a, x)
    pbar = p // bc
    halves = [list(range(0, pbar, 2)), list(range(1, pbar, 2))]
    c = torch.full_like(want, float("nan"))
    for units in halves:
        pl = bs.SttsmPlan(m, n, p, ba, bc, units=units)
        part = torch.full_like(want, float("nan"))
        pl.run(a, x, part)
        idx = torch.as_tensor(pl.c_block_ranks(), device="cuda")
        mask = torch.zeros(want.numel() // bc**m, dtype=torch.bool, device="cuda")
        mask[idx] = True
        assert torch.isnan(part.view(-1, bc**m)[~mask]).all()  # nothing written outside its blocks
        c.view(-1, bc**m)[idx] = part.view(-1, bc**m)[idx]
        pl.close()
    torch.cuda.synchronize()
    assert torch.equal(c, want)
    full_ws = bs.SttsmPlan(m, n, p, ba, bc).workspace_bytes
    pl = bs.SttsmPlan(m, n, p, ba, bc, workspace_limit=full_ws // 3)
    assert pl.stats()["waves"] > 1 and pl.workspace_bytes <= full_ws // 3
    c2 = torch.empty_like(want)
    pl.run(a, x, c2)
    torch.cuda.synchronize()
    assert torch.equal(c2, want)


def test_workspace_fits_free_memory_automatically():
    """With most of HBM taken, the config-5 plan splits its units into waves on
    its own (torch-owned workspace path) and reproduces C bitwise."""
    m, n, p, ba, bc = CFG[5]
    a = random_bcss_device(m, n, ba, 81)
    x = random_matrix_device(p, n, 82)
    want = run(CFG[5], a, x)
    need = bs.SttsmPlan(m, n, p, ba, bc).workspace_bytes
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    budget = 40 << 30                         # leave ~40 GB of the 96 GB the single wave wants
    hog = torch.empty(int(free - budget), dtype=torch.uint8, device="cuda")
    try:
        plan = bs.SttsmPlan(m, n, p, ba, bc)
        c = torch.empty_like(want)
        plan.run(a, x, c)
        torch.cuda.synchronize()
        assert plan.stats()["waves"] > 1 and plan.workspace_bytes < budget < need
        assert torch.equal(c, want)
        plan.close()
    finally:
        del hog
        torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_cascade_is_bitwise_identical_to_level_synchronous(cfg_id, monkeypatch):
    """The cascade (first wave's levels as first-index key groups gated on A
    chunks and upstream groups) reorders launches, not arithmetic: forced on
    and forced off, the pipelined host run returns the same bits."""
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 81 + cfg_id)
    x = random_matrix_device(p, n, 82 + cfg_id)
    a_h, x_h = a.cpu().pin_memory(), x.cpu().pin_memory()
    outs = []
    for env in ("BCSS_FORCE_CASCADE", "BCSS_NO_CASCADE"):
        monkeypatch.setenv(env, "1")
        plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=4)
        plan.stats()  # build with the variable set
        monkeypatch.delenv(env)
        c_h = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
        plan.run_host(a_h.numpy(), x_h.numpy(), c_h.numpy())
        outs.append(c_h.clone())
        plan.close()
    assert torch.equal(outs[0], outs[1])
    assert not torch.isnan(outs[0]).any()


@pytest.mark.parametrize("cfg_id", [2, 3, 4])
def test_noreuse_full_size_matches_reuse(cfg_id):
    """reuse=False (product-keyed temporaries; its top level reads A through
    general mode permutations on the fast kernel) agrees with reuse=True at
    full size to fp64 rounding."""
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 91 + cfg_id)
    x = random_matrix_device(p, n, 92 + cfg_id)
    want = run(CFG[cfg_id], a, x)
    plan = bs.SttsmPlan(m, n, p, ba, bc, reuse=False)
    c = torch.full_like(want, float("nan"))
    plan.run(a, x, c)
    torch.cuda.synchronize()
    assert float((c - want).norm() / want.norm()) <= 1e-13
    plan.close()


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_pipelined_host_run_noreuse(cfg_id):
    """Pipelined host run with reuse=False (product keys: the top level waits
    for all of A instead of key ranges) equals the device run bit for bit."""
    m, n, p, ba, bc = CFG[cfg_id]
    a = random_bcss_device(m, n, ba, 95 + cfg_id)
    x = random_matrix_device(p, n, 96 + cfg_id)
    plan = bs.SttsmPlan(m, n, p, ba, bc, reuse=False, pipeline=3)
    c_dev = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.run(a, x, c_dev)
    torch.cuda.synchronize()
    a_h, x_h = a.cpu().pin_memory(), x.cpu().pin_memory()
    c_h = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(a_h.numpy(), x_h.numpy(), c_h.numpy())
    assert torch.equal(c_h, c_dev.cpu())
    plan.close()


def test_units_run_host_writes_only_own_blocks():
    """A shard plan's host run fills exactly its own C blocks (the rest of the
    caller's buffer is untouched) with the device-path values."""
    m, n, p, ba, bc = CFG[3]
    a = random_bcss_device(m, n, ba, 101)
    x = random_matrix_device(p, n, 102)
    want = run(CFG[3], a, x).cpu().numpy()
    plan = bs.SttsmPlan(m, n, p, ba, bc, units=[0, 5, 11])
    c_h = np.full(plan.c_elems, np.nan)
    plan.run_host(a.cpu().numpy(), x.cpu().numpy(), c_h)
    blk = bc**m
    own = np.zeros(plan.c_elems, dtype=bool)
    for r in plan.c_block_ranks():
        own[r * blk:(r + 1) * blk] = True
    assert np.array_equal(c_h[own], want[own])
    assert np.isnan(c_h[~own]).all()
    plan.close()


@pytest.mark.parametrize("cfg", [(3, 1024, 1024, 32, 32), (6, 48, 48, 8, 8), (5, 128, 64, 16, 8),
                                 (4, 256, 192, 32, 16), (3, 384, 256, 32, 32)])
def test_beyond_baseline_shapes_checksum(cfg):
    """Shapes outside the BASELINE list (bigger n, m = 6, b_a != b_c, p != n,
    non-power-of-two block counts): multilinear checksum on the device path and
    the pipelined host path."""
    m, n, p, ba, bc = cfg
    a = random_bcss_device(m, n, ba, 111)
    x = random_matrix_device(p, n, 112)
    c = run(cfg, a, x)
    v = torch.randn(p, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(9))
    rhs, rhs_abs = multilinear_form(a, m, n, ba, x.t() @ v)
    lhs, lhs_abs = multilinear_form(c, m, p, bc, v)
    assert abs(lhs - rhs) <= 1e-11 * max(lhs_abs, rhs_abs)
    torch.cuda.empty_cache()
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=4)
    c_h = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(a.cpu().pin_memory().numpy(), x.cpu().pin_memory().numpy(), c_h.numpy())
    assert float((c_h.cuda() - c).norm() / c.norm()) <= 1e-13
    plan.close()


def test_pipelined_host_run_refits_workspace_when_hbm_is_short():
    """With most of HBM taken, the pipelined host run re-plans its waves to fit
    the free memory (more waves than modelled) and still returns the same C."""
    m, n, p, ba, bc = CFG[3]
    a = random_bcss_device(m, n, ba, 121)
    x = random_matrix_device(p, n, 122)
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=3)
    c_dev = torch.empty(plan.c_elems, dtype=torch.float64, device="cuda")
    plan.run(a, x, c_dev)
    torch.cuda.synchronize()
    want = c_dev.cpu()
    need = plan.workspace_bytes
    waves0 = plan.stats()["waves"]
    plan.close()
    del c_dev
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    # leave room for A/X/C copies plus ~70 % of the workspace
    keep = 3 * plan.c_elems * 8 + int(0.7 * need)
    hog = torch.empty(max(0, free - keep) // 8, dtype=torch.float64, device="cuda")
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=3)
    c_h = torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(a.cpu().pin_memory().numpy(), x.cpu().pin_memory().numpy(), c_h.numpy())
    assert plan.stats()["waves"] > waves0
    assert torch.equal(c_h, want)
    plan.close()
    del hog


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_async_host_runs_overlap_and_stay_correct(cfg_id):
    """Three streamed host runs with different inputs in flight at once (the
    plan alternates two device buffer sets): every C equals its synchronous
    result bit for bit."""
    m, n, p, ba, bc = CFG[cfg_id]
    plan = bs.SttsmPlan(m, n, p, ba, bc, pipeline=3)
    ins, want = [], []
    for s in range(3):
        a = random_bcss_device(m, n, ba, 131 + s).cpu().pin_memory()
        x = random_matrix_device(p, n, 141 + s).cpu().pin_memory()
        c = torch.empty(plan.c_elems, dtype=torch.float64).pin_memory()
        plan.run_host(a.numpy(), x.numpy(), c.numpy())
        ins.append((a, x))
        want.append(c.clone())
    outs = [torch.full((plan.c_elems,), float("nan"), dtype=torch.float64).pin_memory() for _ in range(3)]
    for (a, x), c in zip(ins, outs):
        plan.run_host_async(a.numpy(), x.numpy(), c.numpy())
    plan.wait()
    for c, w in zip(outs, want):
        assert torch.equal(c, w)
    plan.close()
