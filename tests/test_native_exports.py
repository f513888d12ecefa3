"""CPU checks of the C-ABI library: it loads without a GPU and exports every
symbol include/varstream.h declares; ctypes struct layouts match the header."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "varstream.h"


@pytest.fixture(scope="module")
def lib():
    from paper_2010_02164_b200 import _native

    if not _native.LIB_PATH.exists():
        import __graft_entry__

        __graft_entry__.build()
    return _native.load_library()


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|size_t)\s+(vs_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_bound_exports():
    from paper_2010_02164_b200 import _native

    assert header_functions() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.vs_version() >= 1


def test_struct_layouts_match_header():
    from paper_2010_02164_b200 import _native

    text = HEADER.read_text()
    body = text[text.index("typedef struct vs_state"):text.index("} vs_state;")]
    fields = re.findall(r"\*\s*(\w+);", body)
    assert fields == _native.STATE_FIELDS
    cfg = text[text.index("typedef struct vs_config"):text.index("} vs_config;")]
    names = []
    for decl in re.findall(r"(?:int32_t|double)\s+([\w, ]+);", cfg):
        names += [x.strip() for x in decl.split(",")]
    assert names == [f for f, _ in _native.VsConfig._fields_]
    assert _native.VsConfig.delta.offset == 48 and C.sizeof(_native.VsConfig) == 56


def test_host_argument_errors_map_to_reference_taxonomy(lib):
    from paper_2010_02164_b200 import ConfigError, _native

    rc = lib.vs_row_lse_topm(None, 0, 10, 10, 3, 1, None, 1, None, None, None, None, None)
    assert rc == _native.VS_ERR_CONFIG
    with pytest.raises(ConfigError):
        _native.check(rc, "vs_row_lse_topm")


def test_engine_refuses_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2010_02164_b200 import DecodeConfig, Vocabulary
    from paper_2010_02164_b200.engine import SearchEngine

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        SearchEngine(DecodeConfig(k=2, n=2), Vocabulary(10, 0, 1))


def test_decode_config_validation_matches_reference():
    import math

    from paper_2010_02164_b200 import ConfigError, DecodeConfig

    c = DecodeConfig(k=4, n=3)
    assert c.max_candidates == 4 and c.capacity == 12 and c.delta == math.inf
    for bad in (dict(k=0, n=1), dict(k=2, n=0), dict(k=2, n=1, epsilon=1.0),
                dict(k=2, n=1, delta=-1.0), dict(k=2, n=1, max_candidates=3),
                dict(k=2, n=1, max_len=1), dict(k=2, n=1, capacity=1),
                dict(k=2, n=1, flush_interval=0), dict(k=2, n=1, cost_c0=0, cost_c1=0)):
        with pytest.raises(ConfigError):
            DecodeConfig(**bad)


def test_metrics_rounding_goldens():
    from goldens import load
    from paper_2010_02164_b200 import MetricsReport

    for row in load("metrics.json"):
        r = MetricsReport(timesteps=row["steps"], candidate_expansions=row["expansions"])
        assert r.summarize() == row["summary"]


def test_every_entry_rejects_bad_arguments_before_touching_the_device(lib):
    """Each C-ABI entry validates its host-side arguments first and returns
    VS_ERR_CONFIG (-> ConfigError) without a CUDA call (this runs without a GPU)."""
    from paper_2010_02164_b200 import _native as N

    E = N.VS_ERR_CONFIG
    assert lib.vs_row_lse_topm_ws(None, 0, 10, 10, 3, 1, None, 1, None, None, None, None, None, 0, None) == E
    assert lib.vs_row_attention(None, 64, None, None, 0, 0, None, None, None, None, 0, None, 0, 16, 64,
                                0.125, 1, None, 1, None) == E
    assert lib.vs_row_attention_grouped(None, 64, None, None, 0, 0, None, None, None, None, 1, None, 0, 16,
                                        64, 0.125, None) == E
    assert lib.vs_proj_lse_topm(None, 1024, None, 1024, 1, None, 1, 1024, 100, 5, 2, None, None, 128, None,
                                None, None, None, None, 0, None) == E
    assert lib.vs_rows_copy(None, 0, 1, 0, 16, None, None, 1, None) == E
    assert lib.vs_scatter_rows(None, 0, None, 0, 16, None, None, 1, None) == E
    # head_dim other than 64 is a configuration error even with (dummy) pointers
    buf = C.create_string_buffer(64)
    p = C.addressof(buf)
    assert lib.vs_row_attention_grouped(p, 64, p, p, 0, 0, p, p, p, p, 1, p, 0, 16, 32, 0.125, None) == E


def test_host_materialisation_extension_builds_candidates():
    """_vsmat (hostsrc/vsmat.c) builds real Candidate objects in bulk: the
    append layout (fill) and the packed gather layout (fill_packed)."""
    import numpy as np

    from paper_2010_02164_b200 import _native
    from paper_2010_02164_b200.core import Candidate

    mat = _native.load_vsmat()
    k = 3
    toks = np.array([9, 9, 0, 5, 2, 0, 7, 1, 2, 0, 4], dtype=np.int32)
    count = np.array([2, 1], dtype=np.int32)
    lens = np.array([3, 2, 0, 3, 0, 0], dtype=np.int32)
    offs = np.array([2, 9, 0, 5, 0, 0], dtype=np.int32)
    scores = np.array([-1.5, -2.25, 0, -0.125, 0, 0], dtype=np.float64)
    out = [None] * 4
    mat.fill(out, np.array([3, 1], dtype=np.int64), 0, count, lens, scores, offs, toks, k, Candidate)
    assert out[3] == [Candidate((0, 5, 2), -1.5, True, 3), Candidate((0, 4), -2.25, True, 3)]
    assert out[1] == [Candidate((0, 7, 1), -0.125, True, 1)]
    c = out[3][0]
    assert isinstance(c, Candidate) and hash(c) == hash(Candidate((0, 5, 2), -1.5, True, 3))
    with pytest.raises(Exception):
        c.score = 0.0  # frozen
    out2 = [None] * 2
    mat.fill_packed(out2, np.array([1, 0], dtype=np.int64), np.array([1, 2], dtype=np.int32),
                    np.array([2, 1, 3], dtype=np.int32), np.array([-1.0, -2.0, -3.0]),
                    np.array([0, 4, 0, 0, 6, 2], dtype=np.int32), Candidate)
    assert out2[1] == [Candidate((0, 4), -1.0, True, 1)]
    assert out2[0] == [Candidate((0,), -2.0, True, 0), Candidate((0, 6, 2), -3.0, True, 0)]
    with pytest.raises(ValueError):
        mat.fill(out, None, 0, count, lens, scores, np.array([2, 99, 0, 5, 0, 0], dtype=np.int32), toks, k,
                 Candidate)


def test_host_materialisation_compacted_layout():
    """fill with k = 0: only the emitted candidates' metadata, consecutive."""
    import numpy as np

    from paper_2010_02164_b200 import _native
    from paper_2010_02164_b200.core import Candidate

    mat = _native.load_vsmat()
    toks = np.array([9, 0, 5, 2, 0, 7, 1, 0, 4], dtype=np.int32)
    out = [None] * 2
    mat.fill(out, None, 0, np.array([2, 1], dtype=np.int32), np.array([3, 2, 3], dtype=np.int32),
             np.array([-1.0, -2.0, -3.0]), np.array([1, 7, 4], dtype=np.int32), toks, 0, Candidate)
    assert out[0] == [Candidate((0, 5, 2), -1.0, True, 0), Candidate((0, 4), -2.0, True, 0)]
    assert out[1] == [Candidate((0, 7, 1), -3.0, True, 1)]
    with pytest.raises(ValueError):
        mat.fill(out, None, 0, np.array([3, 1], dtype=np.int32), np.array([3, 2, 3], dtype=np.int32),
                 np.array([-1.0, -2.0, -3.0]), np.array([1, 7, 4], dtype=np.int32), toks, 0, Candidate)
