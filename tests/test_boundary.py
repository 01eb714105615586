"""CPU: the drop-in boundary.  libqvk.so loads and exports every symbol include/qvk.h declares; libqv_prefill.so
exports the whole qv:: API of the reference's prefill.hpp; the host-only parts of the C ABI (group scheduler,
retention arithmetic, validation texts) agree with the reference.  No kernel is launched here."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2505_16175_b200 as qp
from paper_2505_16175_b200 import QvError
from oracle import oracle as O

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2505_16175_b200" / "lib"


def _exports(path: Path) -> set[str]:
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_libqvk_exports_every_header_symbol():
    declared = qp.header_symbols()
    assert len(declared) >= 20
    exported = _exports(LIB / "libqvk.so")
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:  # and they resolve through ctypes
        assert hasattr(qp.lib, s)


def test_libqvk_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB / "libqvk.so")], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB / "libqvk.so")], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM", "STTM"):  # tcgen05.mma / TMA / tcgen05.ld / tcgen05.st
        assert mnemonic in sass, mnemonic


@pytest.mark.skipif(not (LIB / "libqv_prefill.so").exists(), reason="drop-in shim not built")
def test_shim_exports_reference_api():
    demangle = lambda names: set(
        subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines())
    ours = {s for s in demangle(_exports(LIB / "libqv_prefill.so")) if s.startswith("qv::")}
    want = [
        "qv::ModelConfig::validate() const", "qv::PruneConfig::validate() const",
        "qv::scorer_from_name(std::__cxx11::basic_string<char, std::char_traits<char>, std::allocator<char> > const&)",
        "qv::scorer_name(qv::Scorer)", "qv::KvCache::value_bytes() const",
        "qv::KvCache::same_entries(qv::KvCache const&) const", "qv::StandInModel::StandInModel(qv::ModelConfig const&)",
        "qv::StandInModel::patch_grid(unsigned int)", "qv::retained_count(double, unsigned long)",
        "qv::make_cache(qv::ModelConfig const&)", "qv::group_count(unsigned long, unsigned int)",
    ]
    for w in want:
        assert w in ours, w
    for stem in ("qv::StandInModel::tokenize_group(", "qv::StandInModel::tokenize(", "qv::StandInModel::project(",
                 "qv::score_tokens(", "qv::top_k_indices(", "qv::prune_group(", "qv::prefill_group(",
                 "qv::prefill("):
        assert any(s.startswith(stem) for s in ours), stem
    if O.ref is not None:  # every prefill.cpp definition of the reference has a drop-in counterpart
        ref = demangle(_exports(ROOT / "oracle" / "_ref" / "libqvref.so"))
        ref_prefill = {s.replace("qvref::", "qv::") for s in ref if s.startswith("qvref::") and any(
            t in s for t in ("StandInModel", "score_tokens", "retained_count", "top_k_indices", "prune_group",
                             "make_cache", "prefill", "group_count", "KvCache", "ModelConfig", "PruneConfig",
                             "scorer_"))}
        assert ref_prefill - ours == set()


@pytest.mark.parametrize("rho,n", [(0.5, 1), (0.5, 3), (0.5, 5), (0.125, 4), (0.125, 12), (0.1, 4096), (0.3, 10),
                                   (1e-9, 100), (1.0, 7), (0.999999, 10), (0.05, 30)])
def test_retained_count_matches(rho, n):
    assert qp.retained_count(rho, n) == O.retained_count(rho, n)
    if O.ref is not None:
        assert qp.retained_count(rho, n) == O.ref.qvref_retained_count(rho, n)


def test_validation_messages_match_reference():
    for rho in (0.0, -1.0, 1.5, float("nan")):
        with pytest.raises(QvError, match=re.escape("retention ratio must be in (0, 1]")):
            qp.PruneConfig(rho=rho).validate()
        if O.ref is not None:
            assert O.ref.qvref_validate_prune(rho) == -1
            assert O.ref.qvref_last_error().decode() == "retention ratio must be in (0, 1]"
    with pytest.raises(QvError, match="frames_per_group must be >= 1"):
        qp.group_count(10, 0)
    assert qp.group_count(3600, 16) == 225 and qp.group_count(0, 3) == 0
    with pytest.raises(QvError, match="unknown scorer: bogus"):
        qp.scorer_from_name("bogus")
    assert qp.scorer_from_name("attention_score") == qp.Scorer.attention_score
    with pytest.raises(QvError, match="prune: empty group"):
        qp.prune_group(np.zeros(0), np.zeros(0), 0, 1, 1, qp.PruneConfig(rho=0.5))
    with pytest.raises(QvError, match="score: tensor shape mismatch"):
        qp.score_tokens(np.zeros(3), np.zeros(4), 2, 1, 2, qp.Scorer.key_norm_small)
    with pytest.raises(QvError, match="attention_score scorer requires a text query"):
        qp.score_tokens(np.zeros(4), np.zeros(4), 2, 1, 2, qp.Scorer.attention_score)
    with pytest.raises(QvError, match="score: text query shape mismatch"):
        qp.score_tokens(np.zeros(4), np.zeros(4), 2, 1, 2, qp.Scorer.attention_score, np.zeros(3))


@pytest.mark.parametrize("frames,fpg,tpf,rho", [(16, 4, 64, 0.5), (17, 4, 64, 0.5), (3600, 16, 256, 0.5),
                                                (256, 16, 256, 0.25), (1, 1, 1, 1.0), (1024, 64, 64, 0.125)])
def test_plan_matches_oracle(frames, fpg, tpf, rho):
    plan = qp.GroupPlan.plan(frames, fpg, tpf, rho)
    tok, keep, row = O.plan_groups(frames, fpg, tpf, rho)
    assert plan.tok_off.tolist() == tok.tolist()
    assert plan.keep.tolist() == keep.tolist()
    assert plan.row_off.tolist() == row.tolist()
    assert plan.first_token.tolist() == tok[:-1].tolist()  # prefill.cpp:139 first_token = frame_begin * tpf


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("frames,fpg", [(3600, 16), (256, 16), (17, 4), (5, 1), (3, 1)])
def test_rank_partition(world, frames, fpg):
    plan = qp.GroupPlan.plan(frames, fpg, 256, 0.5, world=world)
    rb = plan.rank_begin
    G = plan.n_groups
    assert rb[0] == 0 and rb[-1] == G and (np.diff(rb) >= 0).all()
    if G >= world:
        assert (np.diff(rb) >= 1).all()  # nobody idles while groups remain
    cost = plan.sizes.astype(np.float64) ** 2
    per_rank = [cost[rb[r]:rb[r + 1]].sum() for r in range(world)]
    if G >= 4 * world:
        assert max(per_rank) <= cost.sum() / world + cost.max()  # balanced within one group
    shards = [plan.shard(r, world) for r in range(world)]
    assert sum(s.total_tokens for s in shards) == plan.total_tokens
    assert sum(s.total_rows for s in shards) == plan.total_rows
    for r, s in enumerate(shards):
        assert s.row_base == plan.row_off[rb[r]]
        assert s.first_token.tolist() == plan.first_token[rb[r]:rb[r + 1]].tolist()


def test_plan_errors():
    with pytest.raises(QvError, match="tokenize: frames_per_group must be >= 1"):
        qp.GroupPlan.plan(10, 0, 4, 0.5)
    with pytest.raises(QvError, match="tokenize: empty frame buffer"):
        qp.GroupPlan.plan(0, 4, 4, 0.5)
    with pytest.raises(QvError, match=re.escape("retention ratio must be in (0, 1]")):
        qp.GroupPlan.plan(10, 4, 4, 0.0)


def test_patch_grid_matches_reference():
    for tpf in (1, 2, 4, 6, 64, 100, 256, 255, 7, 12):
        r, c = C.c_uint32(), C.c_uint32()
        qp.lib.qvk_patch_grid(tpf, C.byref(r), C.byref(c))
        if O.ref is not None:
            rr, cc = C.c_uint32(), C.c_uint32()
            O.ref.qvref_patch_grid(tpf, C.byref(rr), C.byref(cc))
            assert (r.value, c.value) == (rr.value, cc.value)
        assert r.value * c.value == tpf


@pytest.mark.parametrize("G", [1, 2, 3, 5, 8, 16, 17, 64, 225])
@pytest.mark.parametrize("chunks", [1, 4, 8, "taper"])
def test_pipeline_chunk_bounds_cover_every_group_once(G, chunks):
    """Host pipeline chunking (pipeline.chunk_bounds): contiguous, non-empty, ascending, covering [0, G) exactly;
    'taper' is symmetric-ish with the smallest chunks at both ends."""
    from paper_2505_16175_b200.pipeline import chunk_bounds
    b = [int(x) for x in chunk_bounds(G, chunks)]
    assert b[0] == 0 and b[-1] == G
    assert all(y > x for x, y in zip(b, b[1:]))
    if chunks == "taper" and len(b) > 3:
        sizes = [y - x for x, y in zip(b, b[1:])]
        assert sizes[0] == min(sizes) and sizes[-1] == min(sizes)


def test_c_abi_rejects_bad_arguments_without_a_gpu():
    """Argument validation of the C ABI runs before any device work (the reference's texts where one exists)."""
    import ctypes as C
    lib = qp.lib
    assert lib.qvk_validate_rho(0.0) == -1 and "retention ratio" in lib.qvk_last_error().decode()
    assert lib.qvk_validate_rho(0.5) == 0
    n = C.c_size_t(0)
    # decode workspace size query is pure host arithmetic; bad shapes are rejected
    assert lib.qvk_decode_workspace(1, 28, 4, 64, 100, C.byref(n)) == -3  # head_dim 64: unsupported
    assert lib.qvk_decode_workspace(1, 27, 4, 128, 100, C.byref(n)) == -1  # n_q not a multiple of n_kv
    assert lib.qvk_decode_workspace(1, 28, 4, 128, 100, C.byref(n)) == 0 and n.value > 0
    assert lib.qvk_ipc_get_handle(None, None, None) == -1


def test_reserve_sms_bounds_and_previous_value():
    """qvk_reserve_sms (host-only bookkeeping: the persistent grids read it at launch) returns the previous
    reservation and rejects n < 0 and n >= the SM count with QVK_E_INVALID and a message."""
    prev = qp.reserve_sms(8)
    try:
        assert qp.reserve_sms(3) == 8
        for bad in (-1, 100000):
            with pytest.raises(qp.QvError, match="reserve_sms"):
                qp.reserve_sms(bad)
        assert qp.reserve_sms(0) == 3
    finally:
        qp.reserve_sms(prev)
