"""Host side of the input codecs: the PFM header parser
and the PNG container checks raise the reference's FormatError messages
(formats.py:55-81, 133-146) before any device work -- goldens from
tests/golden/make_golden_codecs.py."""

import io

import numpy as np
import pytest

from paper_2504_15121_b200 import formats


def test_pfm_header_errors_match_reference(codec_golden):
    for data, msg in codec_golden["pfmerr"]:
        with pytest.raises(formats.FormatError) as ei:
            # every malformed case fails in the header/size checks, before
            # the payload would be copied to a device
            formats.read_pfm_device(data, b"Pf", device="cpu")
        assert str(ei.value) == msg


def test_pfm_header_fields(codec_golden):
    for name, c in codec_golden["pfm"].items():
        magic, w, h, scale, pos = formats._pfm_header(bytes(c["bytes"]))
        ch = int(c["channels"])
        assert (h, w) == c["values"].shape[:2], name
        assert magic == (b"PF" if ch == 3 else b"Pf")
        assert len(c["bytes"]) - pos == w * h * ch * 4
        assert (scale > 0) == name.startswith(("be", "rgb_be"))


def test_png16_container_checks():
    from PIL import Image
    buf = io.BytesIO()
    Image.fromarray(np.zeros((4, 4), np.uint8)).save(buf, format="PNG")
    with pytest.raises(formats.FormatError, match="expected 16-bit single-channel PNG, got mode 'L'"):
        formats._png16_samples(buf.getvalue())
    with pytest.raises(formats.FormatError, match="not a decodable PNG"):
        formats._png16_samples(b"\x89PNG garbage")


def test_png16_samples_golden(codec_golden):
    for name, c in codec_golden["png"].items():
        assert np.array_equal(formats._png16_samples(bytes(c["bytes"])), c["raw"]), name


def test_write_pfm_layout():
    from paper_2504_15121_b200 import ScalarField
    v = np.arange(6, dtype=np.float64).reshape(2, 3)
    v[0, 1] = np.nan
    data = formats.write_pfm(ScalarField.from_array(v))
    assert data.startswith(b"Pf\n3 2\n-1.0\n")
    body = np.frombuffer(data[len(b"Pf\n3 2\n-1.0\n"):], "<f4").reshape(2, 3)
    assert np.array_equal(body[::-1], v.astype(np.float32), equal_nan=True)
