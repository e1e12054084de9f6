"""C ABI (CPU): the shared library loads without a GPU and exports every declared symbol."""

import re
from pathlib import Path

from paper_2605_04550_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    src = (ROOT / "include" / "psb200.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(psb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_exports_list():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.psb_version() == 1


def _struct_fields(name):
    hdr = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "psb200.h").read_text(), flags=re.S)
    body = re.search(r"typedef struct \{([^{}]*)\} " + name + ";", hdr).group(1)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if decl:
            ctype, names = decl.split(None, 1)
            fields += [(ctype, nm.strip()) for nm in names.split(",")]
    return fields


def test_opts_and_stats_layout_match_header():
    import ctypes as C
    width = {"double": 8, "int64_t": 8, "int32_t": 4}
    for cls, name in ((_lib.Opts, "psb_opts"), (_lib.Stats, "psb_stats")):
        fields = _struct_fields(name)
        assert [f for f, _ in cls._fields_] == [nm for _, nm in fields]
        for (pyname, ctype), (cty, _) in zip(cls._fields_, fields):
            assert C.sizeof(ctype) == width[cty], pyname


def test_no_gpu_is_a_loud_failure(monkeypatch):
    """Without a device the handle raises instead of computing anything on the host."""
    import torch
    if torch.cuda.is_available():
        return
    try:
        _lib.Handle(0)
    except _lib.BackendUnavailable:
        return
    raise AssertionError("a handle was created without a CUDA device")
