"""CPU: the C-ABI library loads, exports every symbol include/dattn.h
declares, and validates arguments with the reference's status conventions
(kvsched.h:20-32) before touching a device. No compute call is made here."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2401_02669_b200 as pb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "dattn.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dattn_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    syms = header_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", pb.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # and the python mirror binds every one of them
    assert set(syms) <= set(pb.EXPORTED_SYMBOLS), set(syms) - set(pb.EXPORTED_SYMBOLS)


def test_kvsched_attn_symbols_exported():
    """The drop-in: libdattn.so defines the reference's C++ operator API."""
    out = subprocess.run(["nm", "-DC", "--defined-only", pb.LIB_PATH], capture_output=True, text=True).stdout
    for fn in ["kvsched::attn::compute_micro_attention", "kvsched::attn::combine_partials",
               "kvsched::attn::aggregate_partials", "kvsched::attn::naive_attention",
               "kvsched::attn::multi_head_attention", "kvsched::attn::gqa_kv_head",
               "kvsched::attn::serialize_partial", "kvsched::attn::deserialize_partial",
               "kvsched::attn::AttentionConfig::validate", "kvsched::attn::AttentionConfig::effective_scale",
               "kvsched::attn::KVSegment::validate", "kvsched::attn::AttentionPartial::identity"]:
        assert fn in out, fn


def test_abi_version_and_last_error():
    assert pb.lib.dattn_abi_version() == 1
    assert isinstance(pb.last_error(), str)


def test_null_arguments_are_invalid_argument():
    assert pb.lib.dattn_store_create(None, None) == pb.ERR_INVALID_ARGUMENT
    assert "null" in pb.last_error()
    rep = ctypes.c_void_p()
    ok = ctypes.c_int()
    # test_capi.cpp:131-132: null out-pointer -> INVALID_ARGUMENT
    assert pb.lib.dattn_verify_attention(200, 7, 1e-6, None, ctypes.byref(ok)) == pb.ERR_INVALID_ARGUMENT
    # test_capi.cpp:134: trials = -4 -> INPUT, out-pointers untouched
    assert pb.lib.dattn_verify_attention(-4, 7, 1e-6, ctypes.byref(rep), ctypes.byref(ok)) == pb.ERR_INPUT
    assert rep.value is None


@pytest.mark.parametrize("cfg,err", [
    (dict(head_dim=0, num_q_heads=1, num_kv_heads=1), pb.ContractError),
    (dict(head_dim=8, num_q_heads=3, num_kv_heads=2), pb.ContractError),   # ragged groups
    (dict(head_dim=8, num_q_heads=1, num_kv_heads=1, scale=-1.0), pb.ContractError),
    (dict(head_dim=513, num_q_heads=1, num_kv_heads=1), pb.ContractError),  # above K1g's 512
])
def test_store_config_contract(cfg, err):
    """AttentionConfig::validate (distattention.cpp:39-46) before any CUDA call."""
    with pytest.raises(err):
        pb.Store(**cfg)


def test_host_helpers_match_reference_semantics():
    assert pb.blocks_for_tokens(0, 16) == 0 and pb.blocks_for_tokens(17, 16) == 2
    assert [pb.gqa_kv_head(h, 8, 2) for h in range(8)] == [0, 0, 0, 0, 1, 1, 1, 1]
    with pytest.raises(pb.ContractError):
        pb.gqa_kv_head(4, 4, 4)
    assert pb.effective_scale(64) == 0.125 and pb.effective_scale(64, 0.5) == 0.5
    assert [pb.padded_dim(d) for d in (1, 16, 17, 128, 129, 300)] == [16, 16, 32, 128, 256, 512]


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirror and the C header agree on every struct size/offset."""
    src = tmp_path / "sz.c"
    src.write_text(
        '#include "dattn.h"\n#include <stdio.h>\n#include <stddef.h>\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(dattn_store_config),'
        'sizeof(dattn_range), sizeof(dattn_batch), sizeof(dattn_store_info), sizeof(dattn_stats),'
        'sizeof(dattn_merge_desc), offsetof(dattn_range, tok_begin), offsetof(dattn_batch, scale),'
        'offsetof(dattn_store_config, num_pages)); return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(t) for t in (pb.StoreConfig, pb.Range, pb.Batch, pb.StoreInfo, pb.Stats,
                                       pb.MergeDesc)]
    want += [pb.Range.tok_begin.offset, pb.Batch.scale.offset, pb.StoreConfig.num_pages.offset]
    assert got == want


def test_range_array_packs_like_a_list():
    import paper_2401_02669_b200 as pb
    rs = [pb.Range(3, 0, 5, 77), pb.Range(4, 1, 0, 1000, kv_head=2)]
    a, _ = pb._batch(rs, 2, 0, 0, 0.0)
    b, _ = pb._batch(pb.range_array(rs), 2, 0, 0, 0.0)
    assert a.num_ranges == b.num_ranges == 2
    for i in range(2):
        x, y = a.ranges[i], b.ranges[i]
        assert (x.seq, x.out_row, x.kv_head, x.tok_begin, x.tok_end) == (y.seq, y.out_row, y.kv_head, y.tok_begin, y.tok_end)
    assert pb._batch(pb.range_array([]), 1, 0, 0, 0.0)[0].num_ranges == 0
