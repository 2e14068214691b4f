"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; host-side plan derivation; data model and workloads."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cpsjoin_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"CPSJ_API\s+[\w\s\*]*?\b(cpsj_\w+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    from paper_1707_06814_b200 import _native
    from paper_1707_06814_b200.build import SO, build
    build()
    out = subprocess.run(["nm", "-D", "--defined-only", SO], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (cpsj_\w+)", out))
    declared = header_symbols()
    assert declared, "no declarations parsed"
    assert set(declared) == exported
    assert set(declared) == set(_native.EXPORTS)
    lib = _native.load()
    for name in declared:
        assert hasattr(lib, name)
    assert lib.cpsj_version() >= (1 << 16)


def test_library_is_sm100a():
    from paper_1707_06814_b200.build import SO, build
    build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cuda_means_loud_failure(monkeypatch):
    import torch

    from paper_1707_06814_b200 import _native
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        _native.Context.get()


def reference_flag(dist, mbits, lam, eps):
    # cpsjoin.py:206 and :268 with dist as numpy's uint64 popcount sum
    est = 2.0 * (mbits - np.uint64(dist)) / mbits - 1.0
    return bool(est > (1.0 - eps) * lam)


@pytest.mark.parametrize("ell", [1, 8, 16])
@pytest.mark.parametrize("lam", [0.3, 0.5, 0.6, 0.7, 0.8, 0.9, 0.99])
@pytest.mark.parametrize("eps", [0.0, 0.1, 0.3])
def test_flag_distance_is_the_numpy_rule(ell, lam, eps):
    from paper_1707_06814_b200.cpsjoin import flag_distance
    mbits = 64 * ell
    d = flag_distance(lam, eps, mbits)
    for dist in range(mbits + 1):
        assert reference_flag(dist, mbits, lam, eps) == (dist <= d)


def test_survey_threshold_tables():
    from paper_1707_06814_b200.cpsjoin import CPSJoinParams, make_plan
    acc = {0.5: 144, 0.6: 117, 0.7: 90, 0.8: 63, 0.9: 34}
    flag = {0.5: 140, 0.6: 117, 0.7: 94, 0.8: 71, 0.9: 48}
    for lam in acc:
        p = make_plan(CPSJoinParams(lambda_=lam), 128)
        assert p.accept_dist == acc[lam] and p.flag_dist == flag[lam]
        assert p.split_p == 1.0 / (lam * 128)
    acc16 = {0.5: 279, 0.6: 226, 0.7: 173, 0.8: 118, 0.9: 63}
    for lam in acc16:
        assert make_plan(CPSJoinParams(lambda_=lam, ell=16), 128).accept_dist == acc16[lam]


def test_rep_seeds_prefix_stable():
    from paper_1707_06814_b200.cpsjoin import CPSJoinParams, make_plan
    a = make_plan(CPSJoinParams(lambda_=0.5, repetitions=3, seed=7), 128).rep_seeds
    b = make_plan(CPSJoinParams(lambda_=0.5, repetitions=10, seed=7), 128).rep_seeds
    assert np.array_equal(a, b[:3])


def test_params_validation():
    from paper_1707_06814_b200 import CPSJoinParams
    for kw in [dict(lambda_=1.5), dict(lambda_=0.5, epsilon=1.0), dict(lambda_=0.5, limit=0),
               dict(lambda_=0.5, delta=0.0), dict(lambda_=0.5, repetitions=0), dict(lambda_=0.5, ell=0)]:
        with pytest.raises(ValueError):
            CPSJoinParams(**kw)


def test_hash_stream_matches_oracle():
    from oracle import oracle as O
    from paper_1707_06814_b200.hashing import mix64, uniform_stream, word_stream
    assert int(mix64(0)) == O.mix64(0)
    assert np.array_equal(word_stream(123, 500, offset=17), O.word_stream(123, 500, 17))
    u = uniform_stream(9, 1000)
    assert np.all((u >= 0) & (u <= 1))


def test_dataset_cleaning_semantics():
    from paper_1707_06814_b200 import Dataset
    ds = Dataset.from_token_lists([[5, 3, 3], [7], [3, 5], [9, 8, 1], [100, 200]])
    # [7] dropped (< 2 tokens), second [3, 5] dropped (duplicate), dense remap
    assert len(ds) == 3
    assert [r.tokens.tolist() for r in ds.records] == [[1, 2], [0, 3, 4], [5, 6]]
    assert ds.d == 7
    assert ds.sizes.tolist() == [2, 3, 2]
    ds2 = Dataset.from_token_lists([[5, 3], [9, 8, 1]], d=10)
    assert ds2.records[1].tokens.tolist() == [1, 8, 9]
    assert ds2.csr().shape == (2, 10)
    assert ds2.token_frequency[8] == 1


def test_workload_generator_deterministic_and_planted_exact():
    from paper_1707_06814_b200.workloads import CONFIGS, generate
    a = generate(1, scale=0.02)
    b = generate(1, scale=0.02)
    assert np.array_equal(a.tokens, b.tokens) and np.array_equal(a.offsets, b.offsets)
    lo, hi = CONFIGS[1].j_range
    for s, p in a.planted_pairs[:50]:
        x = set(a.tokens[a.offsets[s]:a.offsets[s + 1]].tolist())
        y = set(a.tokens[a.offsets[p]:a.offsets[p + 1]].tolist())
        assert len(x) == len(y)
        j = len(x & y) / len(x | y)
        assert 0.3 < j < 1.0
    for i in range(a.n):
        row = a.tokens[a.offsets[i]:a.offsets[i + 1]]
        assert np.all(np.diff(row.astype(np.int64)) > 0)
        assert row.max() < a.d


def test_allpairs_prefix_length_spec_examples():
    """SPEC:459-466 examples; the prefix never loses a pair: for every pair of
    sizes with J >= lambda achievable, the two prefixes must overlap."""
    from paper_1707_06814_b200 import prefix_length
    assert prefix_length(10, 0.5) == 6
    assert prefix_length(2, 0.5) == 2
    assert prefix_length(7, 0.999999) == 1
    for lam in (0.3, 0.5, 0.6, 0.7, 0.9):
        prev = 0
        for s in range(1, 300):
            p = prefix_length(s, lam)
            assert 1 <= p <= s and p >= prev      # non-decreasing in |x|
            prev = p
            # overlap needed >= lam |x|: the prefix covers |x| - that + 1
            assert p >= s - int(np.ceil(lam * s)) + 1 - 1e-12
    for s in (5, 50, 500):
        assert [prefix_length(s, lam) for lam in (0.2, 0.4, 0.6, 0.8)] == \
            sorted([prefix_length(s, lam) for lam in (0.2, 0.4, 0.6, 0.8)], reverse=True)
    with pytest.raises(ValueError):
        prefix_length(0, 0.5)


def test_lsh_repetitions_for_recall_spec_examples():
    from paper_1707_06814_b200.lsh import MinHashJoinParams, repetitions_for_recall, rep_plan
    assert repetitions_for_recall(0.5, 4, 0.9) == 37
    assert repetitions_for_recall(0.9, 1, 0.9) == 3
    assert repetitions_for_recall(0.5, 3, 1e-12) == 1
    with pytest.raises(ValueError):
        MinHashJoinParams(lambda_=0.5, phi=1.0)
    with pytest.raises(ValueError):
        MinHashJoinParams(lambda_=0.5, k=0)
    # positions are prefix-stable in L and in range
    p5, s5 = rep_plan(3, 5, 4, 128)
    p9, s9 = rep_plan(3, 9, 4, 128)
    assert np.array_equal(p5, p9[:5]) and np.array_equal(s5, s9[:5])
    assert p9.min() >= 0 and p9.max() < 128


def test_lsh_oracle_plan_restatement_matches_host():
    from oracle import oracle as O
    from paper_1707_06814_b200.lsh import rep_plan
    for seed, L, k in [(0, 3, 10), (7, 40, 3), (123, 2, 1)]:
        p, s = rep_plan(seed, L, k, 128, path=(1,) if seed == 0 else ())
        q, r = O.lsh_rep_plan(seed, L, k, 128, path=(1,) if seed == 0 else ())
        assert np.array_equal(p, q) and np.array_equal(s, r)


def test_write_pairs_format(tmp_path):
    from paper_1707_06814_b200.ingest import write_pairs
    p = tmp_path / "out.txt"
    write_pairs(str(p), [0, 3], [5, 9], [0.5, 2.0 / 3.0])
    assert p.read_text() == "0 5 0.500000\n3 9 0.666667\n"


# ------------------------------------------------------------ ABI guard

ABI_STRUCTS = {"cpsj_inputs": "Inputs", "cpsj_plan": "Plan", "cpsj_lsh_plan": "LshPlan", "cpsj_k1_dsts": "K1Dsts",
               "cpsj_join_stats": "JoinStats", "cpsj_ingest_stats": "IngestStats"}


def test_ctypes_structs_match_header_sizeof(tmp_path):
    """The ctypes declarations have the header's sizeof and field offsets
    (gcc on include/cpsjoin_b200.h), and every parameter struct starts with
    its struct_size guard."""
    import ctypes

    from paper_1707_06814_b200 import _native
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "cpsjoin_b200.h"', "int main(void) {"]
    for c_name, py_name in ABI_STRUCTS.items():
        lines.append(f'printf("{py_name} size %zu\\n", sizeof({c_name}));')
        for f, _ in getattr(_native, py_name)._fields_:
            lines.append(f'printf("{py_name} {f} %zu\\n", offsetof({c_name}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        py_name, what, v = ln.split()
        got[(py_name, what)] = int(v)
    for py_name in ABI_STRUCTS.values():
        cls = getattr(_native, py_name)
        assert got[(py_name, "size")] == ctypes.sizeof(cls), py_name
        for f, _ in cls._fields_:
            assert got[(py_name, f)] == getattr(cls, f).offset, (py_name, f)
    for py_name in ("Inputs", "Plan", "LshPlan", "K1Dsts"):
        cls = getattr(_native, py_name)
        assert cls._fields_[0][0] == "struct_size"
        assert cls().struct_size == ctypes.sizeof(cls)
    lib = _native.load()
    assert lib.cpsj_version() == _native.ABI_VERSION


def _integration_stub() -> str:
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = doc.split("<!-- integration-stub:begin -->")[1].split("<!-- integration-stub:end -->")[0]
    return block.split("```python")[1].split("```")[0]


def test_integration_stub_declares_the_header_structs():
    """The INTEGRATION.md stub's ctypes structs have the header's field
    lists (names and order), so it cannot fall behind cpsjoin_b200.h."""
    import ctypes

    from paper_1707_06814_b200 import _native
    ns = {}
    code = _integration_stub()
    # declarations only: everything before the library is opened
    decl = code.split("lib = ctypes.CDLL")[0]
    rest = code.split("\n", 1)[1]
    structs = rest[rest.index("class Inputs"):rest.index("lib.cpsj_ctx_create")]
    exec(decl + "P, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double\n" + structs,
         ns)
    for stub_name, ours in (("Inputs", _native.Inputs), ("Plan", _native.Plan), ("Stats", _native.JoinStats)):
        cls = ns[stub_name]
        assert [f for f, _ in cls._fields_] == [f for f, _ in ours._fields_]
        assert ctypes.sizeof(cls) == ctypes.sizeof(ours)


def test_reference_shaped_embedded_dataset_matches_reference():
    """tests/refshape.py (the stand-in the GPU integration test hands to the
    INTEGRATION.md stub) carries exactly what the reference's own
    embed_dataset returns in every attribute the stub reads."""
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        pytest.skip("reference not present (GPU box)")
    import sys
    sys.path.insert(0, ref_src)
    try:
        from simjoin.core import Dataset
        from simjoin.embed import EmbeddingParams, embed_dataset
    finally:
        sys.path.remove(ref_src)
    from refshape import from_fixture
    z = np.load(os.path.join(ROOT, "tests", "golden", "planted_small.npz"))
    tok, off = z["tokens"], z["offsets"]
    lists = [tok[off[i]:off[i + 1]].astype(np.int64) for i in range(len(off) - 1)]
    ds = Dataset.from_token_lists(lists, d=int(z["d"]))
    ref = embed_dataset(EmbeddingParams(t=int(z["t"]), seed=int(z["emb_seed"])), ds)
    ours = from_fixture(z)
    assert len(ours) == len(ref) and ours.t == ref.t
    assert np.array_equal(ours.verify_csr.indices, ref.verify_csr.indices)
    assert ours.verify_csr.indices.dtype == ref.verify_csr.indices.dtype
    assert np.array_equal(ours.verify_csr.indptr, ref.verify_csr.indptr)
    assert np.array_equal(ours.sizes, ref.sizes) and ours.sizes.dtype == ref.sizes.dtype
    assert np.array_equal(ours.values, ref.values) and ours.values.dtype == ref.values.dtype
    assert np.array_equal(ours.sketches(8, 5), ref.sketches(8, 5))


@pytest.mark.parametrize("t_copy,t_k1", [(8.2e-3, 11.2e-3), (1.4e-3, 3.4e-3), (12e-3, 30e-3), (8e-3, 4e-3),
                                         (1e-6, 1e-6)])
def test_pipelined_chunk_schedule_is_stall_free(t_copy, t_k1):
    """embed._chunk_fractions: cumulative fractions rise to exactly 1, and
    when K1 is slower than the copy (rho >= growth floor) chunk c + 1 has
    arrived by the time chunk c is hashed: T_copy S_{c+1} <= T_copy S_0 + T_k1 S_c."""
    from paper_1707_06814_b200.embed import _MIN_GROWTH, _chunk_bounds, _chunk_fractions
    S = _chunk_fractions(t_copy, t_k1)
    assert S[-1] == 1.0 and all(b > a for a, b in zip(S, S[1:])) and 0 < S[0] <= 1.0 and len(S) <= 64
    if 0.9 * t_k1 / t_copy >= _MIN_GROWTH:
        for c in range(len(S) - 1):
            assert t_copy * S[c + 1] <= t_copy * S[0] + t_k1 * S[c] + 1e-12
    b = _chunk_bounds(100_000, None, nnz=10_000_000, t=128, ell=8)
    assert b[0] == 0 and b[-1] == 100_000 and np.all(np.diff(b) >= 0)
    # no first chunk below ~2 set pairs per warp, however fast the copy
    b = _chunk_bounds(500_000, None, nnz=150_000_000, t=128, ell=16)
    assert b[1] >= 20_000 and len(b) >= 4
    b = _chunk_bounds(100_000, 4)
    assert list(b) == [0, 12500, 25000, 50000, 100000]
