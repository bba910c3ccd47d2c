"""The `fic` command line (proj/tools/main.cpp) and its bench (proj/tools/bench.cpp), re-hosted
on the B200 library.

    python -m paper_1404_0774_b200 encode  in.pgm out.fic [--n 4 --step 0 --s-bits 5 --o-bits 7
                                           --s-max 1.0 --shadow-eps 0 --workers 1 --chunk 16x16]
    python -m paper_1404_0774_b200 decode  in.fic out.pgm [--scale 1 --iterations 16
                                           --initial mid-gray|black|PATH --convergence-eps -1]
    python -m paper_1404_0774_b200 metrics a.pgm b.pgm
    python -m paper_1404_0774_b200 bench   corpus_dir [--sizes 256,512 --workers-list 1,4
                                           --chunk-list 16x16 --repeats 3 --csv bench.csv --n 4 --step 0]

Same subcommands, options, `key=value` stdout lines and exit codes as main.cpp: 0 on success,
2 for a CodecError (main.cpp:210-212) or a usage error, 1 for anything else (main.cpp:213-216).
The bench writes the reference's CSV schema (bench.hpp:31-32).  Its rows are GPU encodes through
the public API (host image in, host records out, wall clock, minimum over --repeats): the
"gpu" row plays the role of the reference's sequential baseline, and one "gpu" row per
--workers-list entry > 1 checks the FIC1 bytes against it before timing, as bench.cpp:94-97
does for its parallel rows (workers keep their validation but do not change the GPU result).
"""
import argparse
import math
import os
import sys
import time

from . import abi
from .codec import CodecError, CodecParams, decode_traced, encode, psnr, rmse, validate_geometry
from .fic1 import deserialize, serialize
from .pgm import load_pgm, write_pgm

CSV_HEADER = "image,side,impl,workers,chunk,encode_ms,speedup,size_reduction_pct"  # bench.hpp:31-32


def _err(name, detail):
    return CodecError(abi.ERRC_NAMES.index(name) + 1, detail)


def _read(path):
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError:
        raise _err("IoError", "cannot open " + path) from None  # image.cpp:125, format.cpp:189


def _write(path, data):
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError:
        raise _err("IoError", "cannot open " + path + " for writing") from None


def parse_chunk(text):
    """main.cpp:25-41: "W" or "WxH", each >= 1."""
    try:
        if "x" not in text:
            w = h = int(text)
        else:
            a, b = text.split("x", 1)
            w, h = int(a), int(b)
    except ValueError:
        raise _err("BadParams", f"chunk '{text}' is not WxH") from None
    if w < 1 or h < 1:
        raise _err("BadParams", f"chunk '{text}' must be at least 1x1")
    return (w, h)


def parse_int_list(text, what):
    """main.cpp:43-59: comma-separated integers, empty items skipped, at least one."""
    out = []
    for item in text.split(","):
        if not item:
            continue
        try:
            out.append(int(item))
        except ValueError:
            raise _err("BadParams", f"{what} list entry '{item}' is not an integer") from None
    if not out:
        raise _err("BadParams", f"empty {what} list")
    return out


def size_reduction_pct(enc, raw_bytes):
    """format.cpp:201-207: (1 - serialized / raw) * 100."""
    if raw_bytes == 0:
        raise _err("BadParams", "raw size is zero; ratio undefined")
    return (1.0 - len(serialize(enc)) / raw_bytes) * 100.0


def cmd_encode(a):
    img = load_pgm(_read(a.input))
    params = CodecParams(n=a.n, step=a.step, s_bits=a.s_bits, o_bits=a.o_bits, s_max=a.s_max,
                         shadow_eps=a.shadow_eps)
    validate_geometry(img, params)
    chunk = parse_chunk(a.chunk)
    t0 = time.perf_counter()
    enc = encode(img, params, workers=a.workers, chunk=chunk)
    elapsed = (time.perf_counter() - t0) * 1e3
    data = serialize(enc)
    _write(a.output, data)
    print(f"encode_ms={elapsed:.3f}")
    print(f"mappings={len(enc.mappings)}")
    print(f"size_reduction_pct={size_reduction_pct(enc, img.size):.3f}")
    print(f"out_bytes={len(data)}")
    return 0


def cmd_decode(a):
    enc = deserialize(_read(a.input))
    initial = a.initial
    if initial not in ("mid-gray", "black"):
        initial = load_pgm(_read(initial))
    eps = None if a.convergence_eps < 0 else a.convergence_eps
    out, _, runs = decode_traced(enc, scale=a.scale, iterations=a.iterations, initial=initial, convergence_eps=eps)
    _write(a.output, write_pgm(out))
    print(f"iterations={runs}")
    print(f"width={out.shape[1]}")
    print(f"height={out.shape[0]}")
    return 0


def cmd_metrics(a):
    x = load_pgm(_read(a.a))
    y = load_pgm(_read(a.b))
    print(f"rmse={rmse(x, y):.6f}")
    p = psnr(x, y)
    print("psnr=inf" if math.isinf(p) else f"psnr={p:.4f}")
    return 0


def run_bench(corpus_dir, params, workers_list, chunks, sizes=None, repeats=3, csv_path="bench.csv", out=None):
    """bench.cpp:42-117 with GPU rows; returns the records (tuples in CSV column order)."""
    out = sys.stdout if out is None else out
    if not os.path.isdir(corpus_dir):
        raise _err("IoError", corpus_dir + " is not a directory")
    files = sorted(f for f in os.listdir(corpus_dir)
                   if f.endswith(".pgm") and os.path.isfile(os.path.join(corpus_dir, f)))
    if not files:
        raise _err("IoError", "no .pgm files in " + corpus_dir)
    fmt = "{:<20} {:>6} {:<10} {:>7} {:<7} {:>12.3f} {:>8.4f} {:>10.3f}"
    out.write("{:<20} {:>6} {:<10} {:>7} {:<7} {:>12} {:>8} {:>10}\n".format(
        "image", "side", "impl", "workers", "chunk", "encode_ms", "speedup", "reduction%"))
    records = []

    def emit(r):
        out.write(fmt.format(*r) + "\n")
        records.append(r)

    def timed(fn):
        best = float("inf")
        for _ in range(repeats):
            t0 = time.perf_counter()
            fn()
            best = min(best, (time.perf_counter() - t0) * 1e3)
        return best

    for name in files:
        try:
            img = load_pgm(_read(os.path.join(corpus_dir, name)))
            if sizes and img.shape[1] not in sizes:
                continue
            validate_geometry(img, params)
            enc = encode(img, params)
            base_bytes = serialize(enc)
            reduction = size_reduction_pct(enc, img.size)
            base_ms = timed(lambda: encode(img, params))
            for w in workers_list:
                if w <= 1:
                    emit((name, img.shape[1], "gpu", 1, "-", base_ms, 1.0, reduction))
                    continue
                for c in chunks:
                    label = f"{c[0]}x{c[1]}"
                    try:
                        if serialize(encode(img, params, workers=w, chunk=c)) != base_bytes:
                            raise _err("BadParams", "parallel output diverged from sequential")
                        ms = timed(lambda: encode(img, params, workers=w, chunk=c))
                        emit((name, img.shape[1], "gpu", w, label, ms, base_ms / ms, reduction))
                    except Exception as e:  # noqa: BLE001 (bench.cpp:107-110: the row is dropped)
                        out.write(f"# {name} workers={w} chunk={label} failed: {e}\n")
        except Exception as e:  # noqa: BLE001 (bench.cpp:112-114: the image is skipped)
            out.write(f"# {name} skipped: {e}\n")
    try:
        with open(csv_path, "w") as f:
            f.write(CSV_HEADER + "\n")
            for r in records:
                f.write("{},{},{},{},{},{:.3f},{:.4f},{:.3f}\n".format(*r))
    except OSError:
        raise _err("IoError", "cannot open " + csv_path + " for writing") from None
    return records


def cmd_bench(a):
    workers = parse_int_list(a.workers_list, "workers")
    chunks = [parse_chunk(c) for c in a.chunk_list.split(",") if c]
    if not chunks:
        raise _err("BadParams", "empty chunk list")
    sizes = parse_int_list(a.sizes, "sizes") if a.sizes else None
    if a.repeats < 1:
        raise _err("BadParams", "repeats must be >= 1")
    params = CodecParams(n=a.n, step=a.step)
    recs = run_bench(a.corpus, params, workers, chunks, sizes, a.repeats, a.csv)
    print(f"rows={len(recs)}")
    print(f"csv={a.csv}")
    return 0


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit 2 (main.cpp:199-202)
        self.print_usage(sys.stderr)
        sys.stderr.write(f"error: {message}\n")
        raise SystemExit(2)


def parser():
    p = _Parser(prog="fic", description="fic - fractal image codec (PIFS, grayscale PGM), B200 backend")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    e = sub.add_parser("encode", help="Encode a PGM image to a FIC1 file")
    e.add_argument("input")
    e.add_argument("output")
    e.add_argument("--n", type=int, default=4)
    e.add_argument("--step", type=int, default=0)
    e.add_argument("--s-bits", type=int, default=5)
    e.add_argument("--o-bits", type=int, default=7)
    e.add_argument("--s-max", type=float, default=1.0)
    e.add_argument("--shadow-eps", type=float, default=0.0)
    e.add_argument("--workers", type=int, default=1)
    e.add_argument("--chunk", default="16x16")
    d = sub.add_parser("decode", help="Decode a FIC1 file to a PGM image")
    d.add_argument("input")
    d.add_argument("output")
    d.add_argument("--scale", type=int, default=1)
    d.add_argument("--iterations", type=int, default=16)
    d.add_argument("--initial", default="mid-gray")
    d.add_argument("--convergence-eps", type=float, default=-1.0)
    m = sub.add_parser("metrics", help="RMSE and PSNR between two PGM images")
    m.add_argument("a")
    m.add_argument("b")
    b = sub.add_parser("bench", help="Benchmark the encoder over a PGM corpus")
    b.add_argument("corpus")
    b.add_argument("--sizes", default="")
    b.add_argument("--workers-list", default="1,4")
    b.add_argument("--chunk-list", default="16x16")
    b.add_argument("--repeats", type=int, default=3)
    b.add_argument("--csv", default="bench.csv")
    b.add_argument("--n", type=int, default=4)
    b.add_argument("--step", type=int, default=0)
    return p


def main(argv=None):
    a = parser().parse_args(argv)
    try:
        return {"encode": cmd_encode, "decode": cmd_decode, "metrics": cmd_metrics, "bench": cmd_bench}[a.cmd](a)
    except CodecError as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except Exception as e:  # noqa: BLE001 (main.cpp:213-216)
        sys.stderr.write(f"error: {e}\n")
        return 1
