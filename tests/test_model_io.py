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
