"""CLI decode / encode (paper_2306_16699_b200/cli.py) against the oracle's
u8 decode (the reference CLI writes ImageBuffer.as_u8 through Pillow).

Bar: PNG pixels equal the oracle's u8 decode except for at most 1 level on
<= 0.1% of the values (the fp32 decode differs from numpy's only in
summation order, which can flip a round-half-away boundary)."""

import json

import numpy as np
import pytest

from oracle import rinr_oracle as O

pytestmark = pytest.mark.gpu


def _png(path):
    from PIL import Image
    with Image.open(path) as im:
        return np.asarray(im.convert("RGB"))


def test_decode_cli(golden, tmp_path, capsys):
    from paper_2306_16699_b200 import cli
    data = golden("c1_r1")["archive"].tobytes()
    src = tmp_path / "c1.rinr"
    src.write_bytes(data)
    models = O.read_models(data)
    out = tmp_path / "out"
    assert cli.main(["--json", "decode", str(src), "-o", str(out)]) == 0
    lines = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert len(lines) == len(models)
    diff_values = total = 0
    for line, m in zip(lines, models):
        got = _png(line["file"]).astype(int)
        want = O.to_u8(O.decode(m)).astype(int)
        assert got.shape == want.shape == (32, 32, 3)
        d = np.abs(got - want)
        assert d.max() <= 1
        diff_values += int((d > 0).sum())
        total += d.size
    assert diff_values <= 0.001 * total
    # --size and --ids
    ids = [lines[3]["record"], lines[0]["record"]]
    assert cli.main(["--json", "decode", str(src), "-o", str(tmp_path / "o2"), "--size", "8x12",
                     "--ids", ",".join(ids)]) == 0
    sel = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert [s["record"] for s in sel] == [lines[0]["record"], lines[3]["record"]]  # archive order
    assert _png(sel[0]["file"]).shape == (8, 12, 3)
    # errors: unknown id -> exit 2; bad usage -> exit 1
    assert cli.main(["decode", str(src), "-o", str(tmp_path / "o3"), "--ids", "nope"]) == 2
    assert cli.main(["decode", str(src)]) == 1


def test_encode_cli_roundtrip(tmp_path, capsys):
    from PIL import Image

    from paper_2306_16699_b200 import cli
    from transforms_common import smooth_images
    x = smooth_images(3, 32, 32, seed=8)
    d = tmp_path / "imgs"
    d.mkdir()
    for i, im in enumerate(x):
        Image.fromarray(np.floor(im * 255 + 0.5).astype(np.uint8), "RGB").save(d / f"im{i}.png")
    arc = tmp_path / "enc.rinr"
    assert cli.main(["--json", "encode", str(d), "-o", str(arc), "--round1-steps", "200", "--retrain-steps",
                     "50"]) == 0
    recs = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert [r["record"] for r in recs[:3]] == ["im0", "im1", "im2"] and recs[3]["records"] == 3
    out = tmp_path / "dec"
    assert cli.main(["decode", str(arc), "-o", str(out)]) == 0
    for i in range(3):
        got = _png(out / f"im{i}.png").astype(np.float64) / 255.0
        tgt = np.floor(x[i] * 255 + 0.5) / 255.0  # the encoder fitted the 8-bit PNG
        psnr = 10 * np.log10(1 / float(np.mean((got - tgt) ** 2)))
        # the PNG reproduces the encoder's reported PSNR up to 8-bit rounding
        assert abs(psnr - recs[i]["psnr_db"]) < 0.3, (psnr, recs[i]["psnr_db"])
