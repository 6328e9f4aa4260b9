"""The C-ABI library loads and exports every symbol include/rabitq.h declares
(CPU-only: no compute calls); without a GPU the product path fails loudly."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "rabitq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rabitq_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_16007_b200 import _build

    _build.build()
    import paper_2605_16007_b200 as rq

    return rq.lib()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 16
    for n in names:
        assert hasattr(lib, n), n
    import paper_2605_16007_b200 as rq

    assert sorted(rq.EXPORTED) == names


def test_version_and_defaults(lib):
    import paper_2605_16007_b200 as rq

    assert b"sm_100a" in lib.rabitq_version()
    o = rq.BuildOpts()
    lib.rabitq_build_opts_default(ctypes.byref(o))
    assert o.device == -1 and o.kmeans_iters == 0
    s = rq.SearchOpts()
    lib.rabitq_search_opts_default(ctypes.byref(s))
    assert s.scan_path == 0 and s.eps0 == 0.0


def test_struct_layouts_match_header():
    """ctypes mirrors of the C structs: field names in header order."""
    import paper_2605_16007_b200 as rq

    src = open(os.path.join(ROOT, "include", "rabitq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)

    def fields(name):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + name + ";", src, re.S).group(1)
        out = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            for part in decl.split(","):
                part = re.sub(r"\[.*?\]", "", part)
                out.append(re.findall(r"\*?\s*([A-Za-z_0-9]+)\s*$", part.strip())[0])
        return out

    assert [f for f, _ in rq.BuildOpts._fields_] == fields("rabitq_build_opts")
    assert [f for f, _ in rq.SearchOpts._fields_] == fields("rabitq_search_opts")
    assert [f for f, _ in rq.Debug._fields_] == fields("rabitq_debug")
    assert [f for f, _ in rq.IndexInfo._fields_] == fields("rabitq_index_info_t")
    assert [f for f, _ in rq.Export._fields_] == fields("rabitq_export_t")
    assert [f for f, _ in rq.Profile._fields_] == fields("rabitq_profile")


def test_argument_errors_without_gpu(lib):
    """Argument validation runs before any device work; with no device the
    build fails loudly with UNSUPPORTED (no CPU fallback)."""
    import numpy as np
    import torch

    import paper_2605_16007_b200 as rq

    with pytest.raises(rq.RabitqError) as e:
        rq.Index(np.zeros((10, 4), np.float32), nlist=20)
    assert e.value.status == rq.ERR_INVALID_ARGUMENT
    if not torch.cuda.is_available():
        with pytest.raises(rq.RabitqError) as e:
            rq.Index(np.random.rand(100, 4).astype(np.float32), nlist=4)
        assert e.value.status == rq.ERR_UNSUPPORTED
    h = ctypes.c_void_p()
    assert lib.rabitq_search(None, None, 0, 1, 1, 1, None, None) == rq.ERR_INVALID_ARGUMENT
    lib.rabitq_free(None)  # no-op


def _struct_fields(name):
    """Member names, in order, of `typedef struct { ... } name;` in include/rabitq.h."""
    src = open(os.path.join(ROOT, "include", "rabitq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    m = re.search(r"typedef struct \{([^{}]*)\}\s*" + re.escape(name) + r"\s*;", src)
    assert m, name
    names = []
    for decl in m.group(1).split(";"):
        decl = re.sub(r"^const\s+", "", decl.strip())
        if not decl:
            continue
        head, _, rest = decl.partition(" ")
        for part in rest.split(","):
            part = part.strip().lstrip("*").strip()
            names.append(re.sub(r"\[.*\]", "", part).strip())
    return names


@pytest.mark.parametrize("cname,pyname", [("rabitq_search_opts", "SearchOpts"), ("rabitq_profile", "Profile"),
                                          ("rabitq_index_info_t", "IndexInfo")])
def test_binding_structs_match_header(cname, pyname):
    """The ctypes mirrors of the C-ABI structs list the header's members in the
    header's order (an appended field on one side only would shift the rest)."""
    import paper_2605_16007_b200 as rq

    py = [f for f, _ in getattr(rq, pyname)._fields_]
    assert py == _struct_fields(cname), (py, _struct_fields(cname))
