"""The INTEGRATION.md ctypes stub, run verbatim (the block between its
markers) on an object shaped like the reference's EmbeddedDataset
(tests/refshape.py), must reproduce the reference's own cpsjoin_self output
stored in a golden fixture -- the binding a maintainer would add to the
reference package, exercised end to end through the C ABI."""
import os
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def stub():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = doc.split("<!-- integration-stub:begin -->")[1].split("<!-- integration-stub:end -->")[0]
    code = block.split("```python")[1].split("```")[0]
    ns = {}
    cwd = os.getcwd()
    os.chdir(ROOT)  # the stub opens the library by its repo-relative path
    try:
        exec(compile(code, "INTEGRATION.md", "exec"), ns)
    finally:
        os.chdir(cwd)
    return ns


@pytest.mark.parametrize("name", ["planted_small", "planted_880", "dense_cluster"])
def test_integration_stub_reproduces_reference_join(stub, name):
    from refshape import from_fixture
    z = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    emb = from_fixture(z)
    for k in range(int(z["n_joins"])):
        lam, ell, seed, reps, limit, eps, delta, cap = z[f"j{k}_params"].tolist()
        ct_key = f"j{k}_use_count_table"
        params = types.SimpleNamespace(lambda_=lam, ell=int(ell), seed=int(seed), repetitions=int(reps),
                                       limit=int(limit), epsilon=eps, delta=delta, depth_cap=int(cap),
                                       use_count_table=bool(int(z[ct_key])) if ct_key in z.files else False)
        a, b, sims, st = stub["gpu_cpsjoin_self"](emb, params)
        assert np.array_equal(a.astype(np.int64), z[f"j{k}_pair_a"])
        assert np.array_equal(b.astype(np.int64), z[f"j{k}_pair_b"])
        assert np.array_equal(sims, z[f"j{k}_pair_sim"])
        assert [st.pre_candidates, st.candidates, st.results, st.max_depth, st.peak_live_members] == \
            z[f"j{k}_counters"].tolist()


def test_stale_struct_size_is_rejected(stub):
    """A caller whose cpsj_plan is shorter than the library's (the round-1
    stub had 11 fields) gets CPSJ_E_ABI, not a read past its struct."""
    import ctypes
    Plan, Inputs, Stats, lib = stub["Plan"], stub["Inputs"], stub["Stats"], stub["lib"]
    ctx = ctypes.c_void_p()
    assert lib.cpsj_ctx_create(0, ctypes.byref(ctx)) == 0
    inp = Inputs(ctypes.sizeof(Inputs), None, None, None, 0, None, 128, None, 8, None)
    plan = Plan(ctypes.sizeof(Plan) - 16, 0.5, 250, 64, 144, 140, 0.1, None, 0, 0, 0, 0.45, 0, 1, 0)
    st = Stats()
    assert lib.cpsj_self_join(ctx, ctypes.byref(inp), ctypes.byref(plan), ctypes.byref(st), None) == -5
    assert b"struct_size" in lib.cpsj_last_error(ctx)
    lib.cpsj_ctx_destroy(ctx)
