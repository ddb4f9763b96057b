"""word2vec vector files: the C++ writer reproduces the reference's
save_model bytes exactly (text %.6g and binary layouts); load_model / detect_format
round-trip them.  Host-resident rows need no GPU; the device-streamed path is gpu-marked."""

import numpy as np
import pytest

from helpers import load_golden

from paper_1604_04661_b200.corpus import Vocabulary
from paper_1604_04661_b200.model import (EmbeddingModel, ModelFormatError, detect_format,
                                         load_debug, load_model, save_debug, save_model)


def _fixture():
    g = load_golden("io")
    toks = str(g["tokens"]).split("\x00")
    voc = Vocabulary(toks, np.arange(len(toks), 0, -1, dtype=np.int64),
                     {t: i for i, t in enumerate(toks)}, 1)
    return g, EmbeddingModel(g["vecs"], np.zeros_like(g["vecs"])), voc


@pytest.mark.parametrize("binary", [False, True])
def test_writer_bytes_match_reference(tmp_path, binary):
    g, model, voc = _fixture()
    path = str(tmp_path / "v")
    save_model(model, voc, path, binary=binary)
    assert open(path, "rb").read() == g[f"bytes_{int(binary)}"].tobytes()
    assert detect_format(path) is binary
    back, v2 = load_model(path)
    assert v2.tokens == voc.tokens
    if binary:
        assert np.array_equal(back.input_vectors.view(np.uint32), model.input_vectors.view(np.uint32))
    else:
        np.testing.assert_allclose(back.input_vectors, model.input_vectors, rtol=1e-5)
    assert not back.output_vectors.any()


@pytest.mark.parametrize("binary", [False, True])
def test_writer_float64_bytes_match_reference(tmp_path, binary):
    """A float64 model: text formats the float64 value itself (the reference's f"{v:.6g}"
    of model.input_vectors[i]), binary casts to float32 -- both byte-identical."""
    g, _, voc = _fixture()
    v64 = g["vecs64"]
    path = str(tmp_path / "v64")
    save_model(EmbeddingModel(v64, np.zeros_like(v64)), voc, path, binary=binary)
    assert open(path, "rb").read() == g[f"bytes64_{int(binary)}"].tobytes()


def test_errors_and_debug_roundtrip(tmp_path):
    g, model, voc = _fixture()
    bad = tmp_path / "bad"
    bad.write_text("nonsense\n")
    with pytest.raises(ModelFormatError):
        load_model(str(bad))
    short = tmp_path / "short"
    short.write_text("3 2\na 1 2\n")
    with pytest.raises(ModelFormatError):
        load_model(str(short), binary=False)
    with pytest.raises(ValueError):
        save_model(EmbeddingModel(model.input_vectors[:3], model.output_vectors[:3]), voc, str(tmp_path / "x"))
    p = str(tmp_path / "dbg.npz")
    save_debug(model, voc, p)
    m2, v2 = load_debug(p)
    assert np.array_equal(m2.input_vectors, model.input_vectors) and v2.tokens == voc.tokens


@pytest.mark.gpu
def test_device_rows_stream_to_same_bytes(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_04661_b200.model import DeviceModel
    g, model, voc = _fixture()
    dm = DeviceModel.from_host(model)
    for binary in (False, True):
        path = str(tmp_path / f"d{int(binary)}")
        save_model(dm, voc, path, binary=binary)
        assert open(path, "rb").read() == g[f"bytes_{int(binary)}"].tobytes()
    v64 = g["vecs64"]
    dm64 = DeviceModel.from_host(EmbeddingModel(v64, np.zeros_like(v64)))
    for binary in (False, True):
        path = str(tmp_path / f"e{int(binary)}")
        save_model(dm64, voc, path, binary=binary)
        assert open(path, "rb").read() == g[f"bytes64_{int(binary)}"].tobytes()


def _read_cases():
    g = load_golden("read")
    return g, str(g["names"]).split("\x00")


@pytest.mark.parametrize("name", _read_cases()[1])
def test_reader_matches_reference_outcomes(tmp_path, name):
    """The native reader (sgns_vectors_header / sgns_vectors_sniff / sgns_parse_vectors with
    the Python per-row fallback) against the reference's own load_model and detect_format
    on a torture set (tests/golden/make_golden.py gen_read): Python number syntax
    (underscores, inf/nan, fullwidth and Arabic-Indic digits), universal newlines, tabs
    inside fields, blank lines, doubled spaces, duplicate tokens, truncation, malformed
    headers, binary files without newlines or with newline-prefixed tokens, invalid UTF-8."""
    g, _ = _read_cases()
    path = str(tmp_path / name)
    with open(path, "wb") as fh:
        fh.write(g[f"{name}__bytes"].tobytes())
    flag = int(g[f"{name}__binary"])
    binary = None if flag < 0 else bool(flag)
    if f"{name}__sniff" in g:
        assert detect_format(path) is bool(int(g[f"{name}__sniff"]))
    else:
        with pytest.raises(ModelFormatError):
            detect_format(path)
    if f"{name}__error" in g:
        kind, msg = str(g[f"{name}__error"]).split(": ", 1)
        with pytest.raises(Exception) as ei:
            load_model(path, binary)
        assert type(ei.value).__name__ == kind
        if kind != "UnicodeDecodeError":  # byte positions are relative to what was decoded
            assert str(ei.value).replace(path, "<path>") == msg
        return
    model, voc = load_model(path, binary)
    assert voc.tokens == str(g[f"{name}__tokens"]).split("\x00")
    assert np.array_equal(model.input_vectors.view(np.uint32), g[f"{name}__vecs"])
    assert voc.index == {t: i for i, t in enumerate(voc.tokens)}
