"""The C-ABI library loads and exports every symbol include/daso.h declares
(CPU only: no compute calls), plus its host-only helpers and argument checks."""
import os
import re
import subprocess

import pytest

from paper_2104_05588_b200 import _lib as L
import paper_2104_05588_b200 as daso

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "daso.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(daso_\w+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    fns = header_functions()
    for name in ("daso_init", "daso_local_sync", "daso_global_send", "daso_global_merge", "daso_step"):
        assert name in fns


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (daso_\w+)", out))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    lib = L.lib()
    for f in header_functions():
        getattr(lib, f)


def test_binding_covers_every_declared_symbol():
    assert sorted(L.EXPORTED) == header_functions()


def test_library_is_sm100a_and_links_pip_nccl():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "nvidia/nccl/lib/libnccl.so.2" in ldd


def test_status_strings_and_version():
    lib = L.lib()
    assert lib.daso_status_string(L.OK) == b"ok"
    assert lib.daso_status_string(L.ERR_PROTOCOL) == b"protocol error"
    assert b"sm_100a" in lib.daso_version()


def test_padded_numel_and_flat_layout():
    assert daso.daso_padded_numel(25_557_032, 4) == 25_557_248
    assert daso.daso_padded_numel(1000, 2) == 1024
    assert daso.daso_padded_numel(128, 1) == 128
    offs, tot = daso.daso_flat_layout([3, 64, 65, 0, 1], 64)
    assert offs == [0, 64, 128, 256, 256] and tot == 320


def test_unique_id_is_128_random_bytes():
    a, b = daso.daso_get_unique_id(), daso.daso_get_unique_id()
    assert len(a) == 128 and a != b


@pytest.mark.parametrize("world,G,B,S,rank,expect", [
    (4, 3, 4, 1, 0, L.ERR_CONFIG),    # world % G != 0
    (4, 0, 4, 1, 0, L.ERR_CONFIG),    # G < 1
    (4, 2, 0, 0, 0, L.ERR_CONFIG),    # B < 1
    (4, 2, 4, 5, 0, L.ERR_CONFIG),    # S > B
    (4, 2, 4, 1, 4, L.ERR_RANGE),     # rank out of range
    (4, 2, 4, 1, -1, L.ERR_RANGE),
])
def test_init_validation_before_any_device_work(world, G, B, S, rank, expect):
    import ctypes as C
    cfg = L.Config(rank, 0, 0, 1, 64, 0.9, 1e-4, L.WIRE_BF16, L.MODE_FAITHFUL, 1, 0)
    h = C.c_void_p()
    assert L.lib().daso_init(C.byref(h), world, G, B, S, C.byref(cfg), C.c_char_p(b"\0" * 128)) == expect
    assert not h.value


def test_init_rejects_bad_epoch_config_and_enums():
    import ctypes as C
    h = C.c_void_p()
    bad_epochs = L.Config(0, 3, 3, 4, 64, 0.9, 1e-4, L.WIRE_BF16, L.MODE_FAITHFUL, 1, 0)
    assert L.lib().daso_init(C.byref(h), 2, 1, 4, 1, C.byref(bad_epochs), C.c_char_p(b"\0" * 128)) == L.ERR_CONFIG
    bad_wire = L.Config(0, 0, 0, 1, 64, 0.9, 1e-4, 7, L.MODE_FAITHFUL, 1, 0)
    assert L.lib().daso_init(C.byref(h), 2, 1, 4, 1, C.byref(bad_wire), C.c_char_p(b"\0" * 128)) == L.ERR_ARGUMENT
    assert L.lib().daso_init(None, 2, 1, 4, 1, C.byref(bad_wire), None) == L.ERR_ARGUMENT
    bad_exch = L.Config(0, 0, 0, 1, 64, 0.9, 1e-4, L.WIRE_BF16, L.MODE_FUSED, 1, 0, 2)
    assert L.lib().daso_init(C.byref(h), 2, 1, 4, 1, C.byref(bad_exch), C.c_char_p(b"\0" * 128)) == L.ERR_ARGUMENT
    bad_mode = L.Config(0, 0, 0, 1, 64, 0.9, 1e-4, L.WIRE_BF16, 3, 1, 0)
    assert L.lib().daso_init(C.byref(h), 2, 1, 4, 1, C.byref(bad_mode), C.c_char_p(b"\0" * 128)) == L.ERR_ARGUMENT


def test_kernel_entry_points_reject_bad_pointers_without_launching():
    lib = L.lib()
    assert lib.daso_k_update(None, None, None, 8, 0.1, 0.9, 0.0, 1.0, None, 0, None, None) == L.ERR_ARGUMENT
    assert lib.daso_k_update(3, 16, 32, 8, 0.1, 0.9, 0.0, 1.0, None, 0, None, None) == L.ERR_ARGUMENT  # misaligned
    assert lib.daso_k_update(16, 32, 48, 8, 0.1, 0.9, 0.0, 1.0, None, 9, None, None) == L.ERR_ARGUMENT  # bad wire
    assert lib.daso_k_merge(16, 8, None, 8, 2, 1, None, 0, None, None) == L.ERR_ARGUMENT
    assert lib.daso_k_merge(16, 8, 32, 8, 2, 0, None, 0, None, None) == L.ERR_ARGUMENT   # S < 1
    assert lib.daso_k_average(16, 16, 32, 8, 2, 0, None, None) == L.ERR_ARGUMENT       # stride < n


def test_null_ctx_calls_are_argument_errors():
    lib = L.lib()
    assert lib.daso_step(None, 0.1, 0, None, None) == L.ERR_ARGUMENT
    assert lib.daso_local_sync(None, None) == L.ERR_ARGUMENT
    assert lib.daso_global_merge(None, None) == L.ERR_ARGUMENT
    assert lib.daso_finalize(None) == L.OK
    assert lib.daso_last_error(None) == b"null context"


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(L, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(L, "_lib", None)
    with pytest.raises(ImportError):
        L.lib()


def test_bucket_partition_tiles_the_bucket():
    """OverlappedLocalSync's buckets (N2) cover every gradient exactly once, contiguously,
    in backward order."""
    import random
    from paper_2104_05588_b200.daso import bucket_partition
    rnd = random.Random(0)
    for trial in range(200):
        numels = [rnd.randint(1, 5000) for _ in range(rnd.randint(1, 40))]
        offsets, n = daso.daso_flat_layout(numels, 64)
        limit = rnd.randint(1, 20000)
        buckets, ranges = bucket_partition(offsets, numels, n, limit)
        assert sorted(i for b in buckets for i in b) == list(range(len(numels)))
        assert [i for b in buckets for i in b] == list(range(len(numels) - 1, -1, -1))
        end = offsets[-1] + numels[-1]
        pos = end
        for (off, cnt), b in zip(ranges, buckets):          # descending, adjacent ranges
            assert off + cnt == pos and cnt > 0
            pos = off
            assert all(offsets[i] >= off and offsets[i] + numels[i] <= off + cnt for i in b)
        assert pos == 0
        assert all(cnt >= limit for (_, cnt) in ranges[:-1]) or len(ranges) == 1


@pytest.mark.parametrize("world,G,mode,expect", [
    (4, 2, L.MODE_FAITHFUL, L.ERR_CONFIG),   # NCCL node collectives cannot loop back on one GPU
    (4, 2, L.MODE_SHARDED, L.ERR_CONFIG),
    (4, 2, 3, L.ERR_CONFIG),                # not a fused mode at G > 1 (mode 3 no longer exists)
    (2, 1, 3, L.ERR_ARGUMENT),              # no mode 3: the round-1 NVLS variant was removed
    (4, 3, L.MODE_FUSED, L.ERR_CONFIG),      # world % G != 0
    (18, 9, L.MODE_FUSED, L.ERR_CONFIG),     # G > 8 peers
])
def test_vcluster_validation_before_any_device_work(world, G, mode, expect):
    import ctypes as C
    cfg = L.Config(0, 0, 0, 1, 64, 0.9, 1e-4, L.WIRE_BF16, mode, 1, 0)
    h = C.c_void_p()
    assert L.lib().daso_vcluster_create(C.byref(h), world, G, 4, 1, C.byref(cfg), 1000) == expect
    if h.value:
        L.lib().daso_vcluster_destroy(h)
    assert L.lib().daso_vcluster_create(None, 2, 1, 4, 1, C.byref(cfg), 1000) == L.ERR_ARGUMENT
    assert L.lib().daso_vcluster_rank(None, 0) is None
    assert L.lib().daso_vcluster_destroy(None) == L.OK
