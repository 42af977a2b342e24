"""The C-ABI library loads without a GPU, exports every symbol include/xdit_usp.h declares, the
Python binding's ctypes signatures match the header, and the pure-host entry points behave."""
import ctypes
import os
import re

import pytest

import oracle
from paper_2411_01738_b200 import usp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xdit_usp.h")


def header_prototypes():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    protos = {}
    for m in re.finditer(r"XDIT_API\s+[\w\s\*]+?\b(xdit_\w+)\s*\(([^)]*)\)\s*;", src):
        name, params = m.group(1), m.group(2).strip()
        n = 0 if params in ("", "void") else len([p for p in params.split(",") if p.strip()])
        protos[name] = n
    return protos


def test_header_parses():
    protos = header_prototypes()
    assert "xdit_usp_attention" in protos and protos["xdit_usp_attention"] == 14
    assert len(protos) >= 17


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(usp.LIB_PATH)
    for name in header_prototypes():
        assert hasattr(L, name), f"{name} declared in xdit_usp.h but not exported"


def test_binding_signatures_match_header():
    protos = header_prototypes()
    assert set(usp._SIGS) == set(protos), set(usp._SIGS) ^ set(protos)
    for name, (args, _res) in usp._SIGS.items():
        assert len(args) == protos[name], f"{name}: binding has {len(args)} args, header {protos[name]}"


def test_version_and_error_string():
    assert usp.version() >= 100
    assert isinstance(usp.last_error(), str)


@pytest.mark.parametrize("S_txt,S_img,N", [(0, 4096, 8), (333, 4096, 8), (226, 17550, 4), (512, 65536, 8),
                                           (5, 27, 3), (7, 9, 8), (0, 1024, 1)])
def test_shard_matches_oracle(S_txt, S_img, N):
    for g in range(N):
        assert usp.shard(S_txt, S_img, N, g) == oracle.shard(S_txt, S_img, N, g)


def test_shard_errors():
    with pytest.raises(usp.XditError) as e:
        usp.shard(0, 3, 4, 3)
    assert e.value.status == "EMPTY_SHARD"
    with pytest.raises(usp.XditError) as e:
        usp.shard(0, 3, 4, 4)
    assert e.value.status == "INVALID_ARG"


def test_plan_errors():
    with pytest.raises(usp.XditError) as e:
        usp.plan(1, 24, 0, 1024, 64, 16, 1, 0)  # 24 % 16 != 0 ("16 does not divide evenly into 24")
    assert e.value.status in ("DIVISIBILITY", "UNSUPPORTED")
    with pytest.raises(usp.XditError) as e:
        usp.plan(1, 24, 0, 1024, 64, 5, 1, 0)
    assert e.value.status == "DIVISIBILITY"


def test_comm_init_mismatch_is_rejected_without_gpu():
    h = ctypes.c_void_p()
    rc = usp.lib().xdit_comm_init(None, 4, 0, 2, 1, ctypes.byref(h))
    assert rc == 4  # COMM_MISMATCH, before any CUDA/NCCL call
    assert "ulysses*ring" in usp.last_error()


def test_launch_counter_exported():
    assert usp.launch_count() >= 0


def test_missing_extension_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback: without the built library the binding raises instead of computing."""
    monkeypatch.setattr(usp, "_lib", None)
    monkeypatch.setattr(usp, "LIB_PATH", str(tmp_path / "libxdit_usp.so"))
    with pytest.raises(ImportError):
        usp.shard(0, 16, 2, 0)


def test_next_rows_reject_bad_arguments_without_gpu():
    """SURVEY §8(f) NEXT 1-2 entry points validate before touching the device."""
    L = usp.lib()
    assert L.xdit_cfg_combine(None, None, None, 8, 1.0, 0, None) == 1  # INVALID_ARG
    assert L.xdit_cfg_tail(None, None, None, 8, 1.0, 0, None, None) == 1
    assert L.xdit_kv_retain(None, None, None, 1, 1, 1, 1, 0, 64, 0, 0, 0, 2, None) == 1
    assert L.xdit_usp_attention_kv(None, None, None, None, None, None, 1, 1, 0, 1, 64, 1, 1, None, None) == 1
