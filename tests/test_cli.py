"""The `fic` CLI and bench re-hosted on the B200 library (proj/tools/main.cpp, bench.cpp;
SURVEY §8 row F4).  Argument parsing and error mapping run on CPU; encode/decode/bench go
through the GPU library and are marked gpu."""
import os

import numpy as np
import pytest

from paper_1404_0774_b200 import cli
from paper_1404_0774_b200.codec import CodecError, CodecParams, EncodedImage
from paper_1404_0774_b200.fic1 import serialize
from paper_1404_0774_b200.pgm import load_pgm, write_pgm


def test_parse_chunk_and_lists():
    assert cli.parse_chunk("16x16") == (16, 16)
    assert cli.parse_chunk("8") == (8, 8)
    assert cli.parse_chunk("4x2") == (4, 2)
    for bad in ["ax2", "0x4", "3x0", "x"]:
        with pytest.raises(CodecError, match="BadParams"):
            cli.parse_chunk(bad)
    assert cli.parse_int_list("1,4,,8", "workers") == [1, 4, 8]
    with pytest.raises(CodecError, match="BadParams: empty workers list"):
        cli.parse_int_list(",", "workers")
    with pytest.raises(CodecError, match="is not an integer"):
        cli.parse_int_list("1,a", "workers")


def test_metrics_and_exit_codes(tmp_path, capsys):
    a = np.arange(64, dtype=np.uint8).reshape(8, 8)
    b = a.copy()
    b[0, 0] += 3
    pa, pb = tmp_path / "a.pgm", tmp_path / "b.pgm"
    pa.write_bytes(write_pgm(a))
    pb.write_bytes(write_pgm(b))
    assert cli.main(["metrics", str(pa), str(pb)]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == f"rmse={np.sqrt(9 / 64):.6f}"
    assert out[1].startswith("psnr=")
    assert cli.main(["metrics", str(pa), str(pa)]) == 0
    assert capsys.readouterr().out.splitlines()[1] == "psnr=inf"
    # CodecError -> exit 2 with "error: <Name>: <detail>" (main.cpp:210-212)
    assert cli.main(["metrics", str(pa), str(tmp_path / "missing.pgm")]) == 2
    assert "error: IoError: cannot open" in capsys.readouterr().err
    with pytest.raises(SystemExit) as e:  # usage error -> 2 (main.cpp:199-202)
        cli.main(["encode"])
    assert e.value.code == 2
    assert cli.main(["bench", str(tmp_path / "nodir")]) == 2


@pytest.mark.gpu
def test_encode_decode_roundtrip(tmp_path, capsys, oracle):
    img = oracle.smooth_image(64, 64)
    src = tmp_path / "in.pgm"
    src.write_bytes(write_pgm(img))
    fic_path, out_path = tmp_path / "x.fic", tmp_path / "out.pgm"
    assert cli.main(["encode", str(src), str(fic_path), "--n", "4", "--step", "2"]) == 0
    lines = dict(l.split("=", 1) for l in capsys.readouterr().out.splitlines())
    assert int(lines["mappings"]) == (64 // 4) ** 2
    # FIC1 bytes of the oracle's records for the same image and parameters (fic1.serialize
    # is pinned to the reference's bytes in test_host.py)
    maps, _ = oracle.encode(img, dict(n=4, step=2))
    want = serialize(EncodedImage(64, 64, CodecParams(n=4, step=2), maps))
    assert fic_path.read_bytes() == want
    assert int(lines["out_bytes"]) == os.path.getsize(fic_path)
    assert cli.main(["decode", str(fic_path), str(out_path), "--iterations", "10", "--scale", "2"]) == 0
    lines = dict(l.split("=", 1) for l in capsys.readouterr().out.splitlines())
    assert lines == {"iterations": "10", "width": "128", "height": "128"}
    got = load_pgm(out_path.read_bytes())
    want, _, _ = oracle.decode(maps, 64, dict(n=4, step=2), 2, 10)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_bench_csv(tmp_path, capsys, oracle):
    corpus = tmp_path / "corpus"
    corpus.mkdir()
    (corpus / "a.pgm").write_bytes(write_pgm(oracle.noise_image(32, 7)))
    (corpus / "b.pgm").write_bytes(write_pgm(oracle.smooth_image(64, 3)))
    (corpus / "bad.pgm").write_bytes(write_pgm(np.zeros((8, 16), np.uint8)))  # not square: skipped
    csv = tmp_path / "bench.csv"
    assert cli.main(["bench", str(corpus), "--workers-list", "1,4", "--repeats", "1", "--csv", str(csv)]) == 0
    out = capsys.readouterr().out
    assert "# bad.pgm skipped: NotSquare" in out
    rows = csv.read_text().splitlines()
    assert rows[0] == cli.CSV_HEADER
    assert len(rows) == 1 + 4
    assert rows[1].startswith("a.pgm,32,gpu,1,-,")
    assert rows[2].startswith("a.pgm,32,gpu,4,16x16,")
