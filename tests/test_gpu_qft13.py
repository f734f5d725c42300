"""The 2^13-amplitude-tile QFT / H pass (k_qft13, round 2) against the oracle's
gate-by-gate circuit and H_n: every
block size it takes (5..10 wires), forward and inverse, sub-ranges, the block
partitions of the default plan and explicit ones (QSIM_QFT_BLOCKS), in-place
(Hadamard, sharded) and block-move (single-GPU QFT) layouts, and the kernel
record proving the pass ran."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_quant_ph_0201042_b200.qsim")

TOL = 1e-10


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def run(n, op, lo, m, inverse=False, world=1, blocks=None, force=True):
    """op on a seeded state; force: QSIM_FORCE_QFT13 (the 13-bit passes even
    where the default plan keeps the 12-bit kernel, i.e. where they do not
    save a pass -- this module tests the kernel at every size)."""
    psi = rand_state(n, 3 * n + lo + 7 * m)
    if blocks:
        os.environ["QSIM_QFT_BLOCKS"] = blocks
    if force:
        os.environ["QSIM_FORCE_QFT13"] = "1"
    try:
        h = Q.qsim_create(n, world)
        Q.qsim_set_state(h, 0, psi)
        Q.qsim_profile(h, True)
        if op == "qft":
            Q.qsim_qft(h, lo, m, inverse)
        elif op == "fft":
            Q.qsim_fft(h, lo, m, inverse)
        else:
            Q.qsim_hadamard(h, lo, m)
        prof = Q.qsim_profile_json(h)
        Q.qsim_profile(h, False)
        got = Q.qsim_get_state(h, 0, 1 << n)
        norm = Q.qsim_norm(h)
        Q.qsim_destroy(h)
    finally:
        os.environ.pop("QSIM_QFT_BLOCKS", None)
        os.environ.pop("QSIM_FORCE_QFT13", None)
    ref = psi.copy()
    if op == "had":
        O.hadamard_range(ref, lo, m)
    else:
        O.qft(ref, lo, m, inverse)
    return got, ref, norm, prof


@pytest.mark.parametrize("inverse", [False, True])
@pytest.mark.parametrize("n,lo,m", [(15, 0, 15), (16, 0, 16), (18, 0, 18), (20, 0, 20), (21, 0, 21),
                                    (22, 0, 22), (23, 0, 23), (24, 0, 24), (20, 2, 15), (19, 4, 10),
                                    (22, 1, 20), (17, 0, 11)])
def test_qft13_default_plan(n, lo, m, inverse):
    got, ref, norm, prof = run(n, "qft", lo, m, inverse)
    assert "k_qft13" in prof, prof.keys()
    assert np.max(np.abs(got - ref)) < TOL
    assert abs(norm - 1) < 1e-12


@pytest.mark.parametrize("n", [15, 16, 17, 20, 21, 24, 25, 28])
def test_default_plan_uses_qft13_where_it_saves_a_pass(n):
    """Default plan: the 13-bit passes exactly where ceil(m/10) < ceil(m/8)
    (a 12-bit pass of <= 8 wires streams faster)."""
    got, ref, _, prof = run(n, "qft", 0, n, False, force=False) if n <= 24 else (None, None, None, None)
    if n > 24:   # large: kernel record only
        h = Q.qsim_create(n)
        try:
            Q.qsim_init_gaussian(h, 1)
            Q.qsim_profile(h, True)
            Q.qsim_qft(h, 0, n, False)
            prof = Q.qsim_profile_json(h)
        finally:
            Q.qsim_destroy(h)
    else:
        assert np.max(np.abs(got - ref)) < TOL
    saves = (n + 9) // 10 < (n + 7) // 8
    assert ("k_qft13" in prof) == saves, (n, prof.keys())


@pytest.mark.parametrize("blocks", ["10,10", "5,10,5", "6,7,7", "9,5,6", "8,6,6", "10,5,5", "7,6,7"])
def test_qft13_block_partitions(blocks):
    n = 20
    got, ref, _, prof = run(n, "qft", 0, n, False, blocks=blocks)
    assert "k_qft13" in prof
    assert np.max(np.abs(got - ref)) < TOL


@pytest.mark.parametrize("n,lo,m", [(22, 0, 22), (20, 0, 20), (21, 3, 12), (24, 0, 24), (22, 2, 18)])
def test_hadamard13(n, lo, m):
    got, ref, _, prof = run(n, "had", lo, m)
    assert "k_qft13" in prof
    assert np.max(np.abs(got - ref)) < TOL


@pytest.mark.parametrize("n,lo,m,inverse", [(20, 0, 20, False), (19, 2, 14, True)])
def test_fft13(n, lo, m, inverse):
    got, ref, _, prof = run(n, "fft", lo, m, inverse)
    assert "k_qft13" in prof
    assert np.max(np.abs(got - ref)) < TOL


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("op", ["qft", "had"])
def test_qft13_sharded(world, op):
    n = 19
    got, ref, _, prof = run(n, op, 0, n, False, world=world)
    assert np.max(np.abs(got - ref)) < TOL


def test_qft13_off_matches_on():
    """QSIM_NO_QFT13 (the 12-bit kernels) and the 13-bit plan agree."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]);"
        "from paper_quant_ph_0201042_b200 import qsim as Q;"
        "h = Q.qsim_create(22); Q.qsim_init_gaussian(h, 3); Q.qsim_qft(h, 0, 22, False);"
        "np.save(sys.argv[2], Q.qsim_get_state(h, 0, 1 << 22))")
    outs = []
    for env in ({}, {"QSIM_NO_QFT13": "1"}):
        path = f"/tmp/qft13_{len(env)}.npy"
        r = subprocess.run([sys.executable, "-c", script, root, path], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append(np.load(path))
    assert np.max(np.abs(outs[0] - outs[1])) < 1e-13


@pytest.mark.parametrize("world,n", [(2, 17), (4, 18), (2, 20), (4, 19)])
@pytest.mark.parametrize("op,inverse", [("qft", False), ("qft", True), ("had", False), ("fft", False)])
def test_rank_group_pass(world, n, op, inverse):
    """Blocks whose wires sit on rank bits run as one k_qft13 rank-group pass
    over peer memory (no shard exchange): the whole-register transform of a
    sharded handle equals the oracle, and rank 0 records no exchange."""
    psi = rand_state(n, 11 * n + world)
    h = Q.qsim_create(n, world)
    try:
        Q.qsim_set_state(h, 0, psi)
        Q.qsim_profile(h, True)
        if op == "qft":
            Q.qsim_qft(h, 0, n, inverse)
        elif op == "fft":
            Q.qsim_fft(h, 0, n, inverse)
        else:
            Q.qsim_hadamard(h, 0, n)
        prof = Q.qsim_profile_json(h)
        Q.qsim_profile(h, False)
        got = Q.qsim_get_state(h, 0, 1 << n)
    finally:
        Q.qsim_destroy(h)
    ref = psi.copy()
    if op == "had":
        O.hadamard_range(ref, 0, n)
    else:
        O.qft(ref, 0, n, inverse)
    assert "k_qft13" in prof, prof.keys()
    assert "group_pair_exchange" not in prof, prof.keys()
    assert np.max(np.abs(got - ref)) < TOL


def test_rank_group_pass_off_matches_on():
    """QSIM_NO_RANK_GROUP_PASS (exchanges, then local passes) and the
    rank-group pass give the same state (world 2 and 8: 8 ranks put three
    wires on rank bits, the block falls back to exchanges)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]);"
        "from paper_quant_ph_0201042_b200 import qsim as Q;"
        "out = [];"
        "exec(\"for w in (2, 8):\\n h = Q.qsim_create(19, w); Q.qsim_init_gaussian(h, 3); Q.qsim_qft(h, 0, 19, False);"
        " Q.qsim_hadamard(h, 2, 15); out.append(Q.qsim_get_state(h, 0, 1 << 19)); Q.qsim_destroy(h)\");"
        "np.save(sys.argv[2], np.stack(out))")
    res = []
    for env in ({}, {"QSIM_NO_RANK_GROUP_PASS": "1"}):
        path = f"/tmp/rgp_{len(env)}.npy"
        r = subprocess.run([sys.executable, "-c", script, root, path], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        res.append(np.load(path))
    assert np.max(np.abs(res[0] - res[1])) < 1e-13


@pytest.mark.parametrize("n,lo,m", [(26, 0, 26), (28, 0, 28), (24, 2, 20), (25, 0, 21), (27, 3, 24)])
def test_hadamard_free_layouts(n, lo, m):
    """H_m with free intermediate layouts (R42: every pass but the last writes
    its tile contiguously, the last puts every bit back) against the oracle;
    at n = 28 every pass is a 13-bit pass."""
    got, ref, norm, prof = run(n, "had", lo, m, force=False)
    assert np.max(np.abs(got - ref)) < TOL
    assert abs(norm - 1) < 1e-12
    if (n, lo, m) == (28, 0, 28):
        assert set(prof) - {"_launches"} == {"k_qft13"}, prof.keys()


def test_hadamard_free_layouts_off_matches_on_and_relabelled_start():
    """QSIM_NO_HFLEX (in-place passes) and the free-layout plan agree, also
    when the register starts in a relabelled layout (a QFT whose closing
    swaps were a relabel: QSIM_NO_BLOCK_MOVES)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]);"
        "from paper_quant_ph_0201042_b200 import qsim as Q;"
        "h = Q.qsim_create(26); Q.qsim_init_gaussian(h, 5); Q.qsim_qft(h, 0, 26, False);"
        "Q.qsim_hadamard(h, 0, 26); Q.qsim_hadamard(h, 1, 22);"
        "np.save(sys.argv[2], Q.qsim_get_state(h, 0, 1 << 26))")
    outs = []
    for env in ({}, {"QSIM_NO_HFLEX": "1"}, {"QSIM_NO_BLOCK_MOVES": "1"}):
        path = f"/tmp/hflex_{len(outs)}.npy"
        r = subprocess.run([sys.executable, "-c", script, root, path], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append(np.load(path))
    assert np.max(np.abs(outs[0] - outs[1])) < 1e-13
    assert np.max(np.abs(outs[0] - outs[2])) < 1e-13


@pytest.mark.parametrize("n,lo,m,inverse", [(24, 0, 20, True), (26, 2, 20, False), (25, 1, 17, True), (23, 0, 18, False)])
def test_qft_sub_register_free_layouts(n, lo, m, inverse):
    """The QFT of a sub-register above position 0 (configs[3]'s inverse QFT on
    the exponent register) with free intermediate layouts against the oracle's
    circuit, and against the block-move plan (QSIM_NO_QFLEX) in a subprocess."""
    got, ref, norm, prof = run(n, "qft", lo, m, inverse, force=False)
    assert np.max(np.abs(got - ref)) < TOL
    assert abs(norm - 1) < 1e-12
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]);"
        "from paper_quant_ph_0201042_b200 import qsim as Q;"
        f"h = Q.qsim_create({n}); Q.qsim_init_gaussian(h, 9); Q.qsim_qft(h, {lo}, {m}, {inverse});"
        f"np.save(sys.argv[2], Q.qsim_get_state(h, 0, 1 << {n}))")
    outs = []
    for env in ({}, {"QSIM_NO_QFLEX": "1"}):
        path = f"/tmp/qflex_{len(outs)}.npy"
        r = subprocess.run([sys.executable, "-c", script, root, path], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append(np.load(path))
    assert np.max(np.abs(outs[0] - outs[1])) < 1e-13


@pytest.mark.parametrize("op,n,lo,m,decline", [("had", 26, 0, 26, 1), ("had", 26, 0, 26, 2), ("qft", 25, 0, 20, 1)])
def test_free_layout_plan_falls_back_part_way(op, n, lo, m, decline):
    """A free-layout plan whose k-th 13-bit pass is declined (test hook
    QSIM_TEST_Q13_DECLINE) finishes in place on the current layout and puts
    every bit back with one permutation pass: the result still equals the
    oracle."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    call = f"Q.qsim_hadamard(h, {lo}, {m})" if op == "had" else f"Q.qsim_qft(h, {lo}, {m}, True)"
    script = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1]);"
        "from paper_quant_ph_0201042_b200 import qsim as Q;"
        f"h = Q.qsim_create({n}); Q.qsim_init_gaussian(h, 4); Q.qsim_profile(h, True); {call};"
        "print(sorted(k for k in Q.qsim_profile_json(h) if not k.startswith('_')));"
        f"np.save(sys.argv[2], Q.qsim_get_state(h, 0, 1 << {n}))")
    path = "/tmp/decline.npy"
    r = subprocess.run([sys.executable, "-c", script, root, path],
                       env=dict(os.environ, QSIM_TEST_Q13_DECLINE=str(decline)),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = np.load(path)
    import ast
    kernels = ast.literal_eval(r.stdout.strip().splitlines()[-1])
    assert "k_qft13" in kernels and len(kernels) > 1, kernels   # the fall-back pass / restore ran
    h = Q.qsim_create(n)
    try:
        Q.qsim_init_gaussian(h, 4)
        psi = Q.qsim_get_state(h, 0, 1 << n)
    finally:
        Q.qsim_destroy(h)
    ref = psi.copy()
    if op == "had":
        O.hadamard_range(ref, lo, m)
    else:
        O.qft(ref, lo, m, True)
    assert np.max(np.abs(got - ref)) < TOL, r.stdout
