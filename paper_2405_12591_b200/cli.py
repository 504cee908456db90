"""Command line for the write / read path on the device.

    python -m paper_2405_12591_b200.cli quantize --input m.dqt --bits 4 [--n 2] --out m.dqz
    python -m paper_2405_12591_b200.cli dequantize --input m.dqz --out m.dqt
    python -m paper_2405_12591_b200.cli import-raw --input m.f32 --rows R --cols C --out m.dqt

The reference's ``quantize`` / ``dequantize`` / ``import-raw`` subcommands (cli.py:44-76,
172-185) with the same flags, exit codes (0 ok, 2 malformed input or usage, 3 invalid
parameters, 4 unknown subcommand) and JSON summary line; the compute is the device path
(``deco_quantize`` = K3, ``deco_dequantize`` = K4) and the files are the byte-compatible
DQT1 / DQZ1 formats.  The analysis subcommands (``bench``, ``analyze-outliers``, ``kv-sim``)
and their CSV writers stay out of scope.
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from . import formats
from .compress import compression_report, deco_dequantize, deco_quantize
from .errors import DquantError, MalformedFile
from .quantize import SUPPORTED_BITS

EXIT_OK, EXIT_MALFORMED, EXIT_BAD_PARAMS, EXIT_UNKNOWN = 0, 2, 3, 4


def _emit(obj):
    sys.stdout.write(json.dumps(obj, sort_keys=True) + "\n")


def _fail(code, message):
    sys.stderr.write(f"error: {message}\n")
    return code


def _read_float_matrix(path):
    t = formats.read_tensor(path)
    if not isinstance(t, np.ndarray):
        raise MalformedFile("expected a float tensor, found a packed one")
    if t.ndim != 2:
        raise MalformedFile(f"expected a 2-D tensor, got {t.ndim}-D")
    return t


def cmd_quantize(args):
    if args.bits not in SUPPORTED_BITS:
        return _fail(EXIT_BAD_PARAMS, f"unsupported bits {args.bits}")
    if args.n < 2:
        return _fail(EXIT_BAD_PARAMS, "decomposition length must be >= 2")
    try:
        m = _read_float_matrix(args.input)
    except (MalformedFile, OSError) as exc:
        return _fail(EXIT_MALFORMED, str(exc))
    q = deco_quantize(m, args.bits, args.n)
    formats.write_mpo(args.out, q)
    rep = compression_report(q)
    _emit({"ratio": rep.ratio, "bytes_original": rep.bytes_original, "bytes_compressed": rep.bytes_compressed,
           "bits": args.bits, "n": args.n})
    return EXIT_OK


def cmd_dequantize(args):
    try:
        q = formats.read_mpo(args.input)
    except (MalformedFile, OSError) as exc:
        return _fail(EXIT_MALFORMED, str(exc))
    out = deco_dequantize(q)
    formats.write_tensor(args.out, out.cpu().numpy() if hasattr(out, "cpu") else out)
    return EXIT_OK


def cmd_import_raw(args):
    if args.rows < 1 or args.cols < 1:
        return _fail(EXIT_BAD_PARAMS, "rows and cols must be >= 1")
    try:
        raw = np.fromfile(args.input, dtype="<f4")
    except OSError as exc:
        return _fail(EXIT_MALFORMED, str(exc))
    if raw.size != args.rows * args.cols:
        return _fail(EXIT_MALFORMED, f"file holds {raw.size} float32 values, expected {args.rows * args.cols}")
    formats.write_tensor(args.out, raw.reshape(args.rows, args.cols))
    return EXIT_OK


def _parsers():
    ps = {}
    p = argparse.ArgumentParser(prog="dquant quantize")
    p.add_argument("--input", required=True)
    p.add_argument("--bits", type=int, required=True)
    p.add_argument("--n", type=int, default=2)
    p.add_argument("--out", required=True)
    ps["quantize"] = (p, cmd_quantize)
    p = argparse.ArgumentParser(prog="dquant dequantize")
    p.add_argument("--input", required=True)
    p.add_argument("--out", required=True)
    ps["dequantize"] = (p, cmd_dequantize)
    p = argparse.ArgumentParser(prog="dquant import-raw")
    p.add_argument("--input", required=True)
    p.add_argument("--rows", type=int, required=True)
    p.add_argument("--cols", type=int, required=True)
    p.add_argument("--out", required=True)
    ps["import-raw"] = (p, cmd_import_raw)
    return ps


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    ps = _parsers()
    if not argv or argv[0] in ("-h", "--help"):
        sys.stderr.write("usage: dquant {" + ",".join(ps) + "} [options]\n")
        return EXIT_OK if argv else EXIT_UNKNOWN
    name, rest = argv[0], argv[1:]
    if name not in ps:
        return _fail(EXIT_UNKNOWN, f"unknown subcommand {name!r}")
    parser, handler = ps[name]
    try:
        args = parser.parse_args(rest)
    except SystemExit as exc:
        return EXIT_MALFORMED if exc.code else EXIT_OK
    try:
        return handler(args)
    except MalformedFile as exc:
        return _fail(EXIT_MALFORMED, str(exc))
    except DquantError as exc:
        return _fail(EXIT_BAD_PARAMS, str(exc))


if __name__ == "__main__":
    sys.exit(main())
