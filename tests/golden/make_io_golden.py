"""Generate tests/golden/io/ from the REFERENCE ITSELF (oracle/_ref): the pin
for the C++ host API's I/O and generators.

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_io_golden.py

Inputs are written here (our own small files, no dataset); every expected
output -- canonical re-saves, model bytes, metrics CSV bytes, generator
output, error class and message -- is produced by the reference library
through oracle/ref_bridge.cpp.  tests/cpp/test_sptucker.cpp (--golden DIR)
replays every line of io/cases.txt against libsptucker_b200.so;
tests/test_io_golden.py re-runs this generator and diffs it when the
reference is present.

cases.txt: one case per line, TAB-separated, kind first:
  load     file order skip_header zero_replace zero_repl override code dims saved message
  model    file code resaved message
  modelgen dims J R mean sd seed file
  mwrite   file comments(|-joined) rows(;-joined, fields ,-joined, %a hex)
  mparse   file code nrows comments(|-joined) message
  planted  dims tJ tR nnz noise tmean tsd seed file
  ratings  dims tJ tR nnz tmean tsd seed target_mean target_sd noise half min max file
  index    dims coord mode code col vec inv message
Lists are comma-joined, '-' means none.  Messages are relative to the
fixture directory (the generator and the replay both run there).
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle_py as O  # noqa: E402

u32p = O.u32p
f64p = O.f64p


def lib():
    L = O.ref()
    vp, ip = C.c_void_p, C.POINTER(C.c_int)
    L.ref_last_message.restype = C.c_char_p
    L.ref_tensor_load_delimited.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.c_double, C.c_size_t,
                                            u32p, ip]
    L.ref_tensor_load_delimited.restype = vp
    L.ref_tensor_save_delimited.argtypes = [vp, C.c_char_p]
    L.ref_tensor_get.argtypes = [vp, u32p, C.POINTER(C.c_size_t), C.c_void_p, C.c_void_p]
    L.ref_model_save.argtypes = [vp, C.c_char_p]
    L.ref_model_load.argtypes = [C.c_char_p, ip, u32p, u32p, C.POINTER(C.c_uint32), ip]
    L.ref_model_load.restype = vp
    L.ref_write_metrics_csv.argtypes = [C.c_char_p, C.c_size_t, f64p, C.c_char_p]
    L.ref_parse_metrics_csv.argtypes = [C.c_char_p, C.c_size_t, f64p, C.POINTER(C.c_size_t), C.c_char_p,
                                        C.c_size_t]
    L.ref_synth_ratings.argtypes = [C.c_int, u32p, u32p, C.c_uint32, C.c_size_t, C.c_double, C.c_double,
                                    C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_int, C.c_double,
                                    C.c_double, u32p, f64p]
    L.ref_indexing.argtypes = [C.c_int, u32p, u32p, C.c_size_t, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                               u32p]
    return L


def msg(L) -> str:
    return L.ref_last_message().decode()


def joined(xs) -> str:
    xs = list(xs)
    return ",".join(str(int(x)) for x in xs) if xs else "-"


# ---- inputs for the delimited reader (written here, small, synthetic) ------
LOAD_INPUTS = {
    "basic.tns": b"1 2 3 1.5\n2 1 1 -0.25\n3 3 2 7\n",
    "separators.tns": b"# comment line\n\n  1,2,3,1.5\r\n2\t1\t1\t-0.25\n\t# indented comment\n3 ,3, 2 ,7e-3\n4 1 1 .5",
    "header.csv": b"# produced by hand\nuser,item,time,rating\n1,1,1,4\n2,3,1,5\n1,2,2,3.5\n",
    "header_only.csv": b"i j k v\n",
    "zero.tns": b"1 1 1 0\n2 2 2 -0\n3 1 2 1\n",
    "override.tns": b"1 1 1 1\n2 2 2 2\n",
    "bad_fields.tns": b"1 1 1 1\n2 2 2\n",
    "bad_fields_extra.tns": b"1 1 1 1 1\n",
    "bad_index_zero.tns": b"1 1 1 1\n0 1 1 1\n",
    "bad_index_alpha.tns": b"1 x 1 1\n",
    "bad_index_frac.tns": b"1 1 1.5 1\n",
    "bad_index_plus.tns": b"+1 1 1 1\n",
    "bad_index_overflow.tns": b"4294967296 1 1 1\n",
    "bad_index_neg.tns": b"-1 1 1 1\n",
    "bad_value_nan.tns": b"1 1 1 nan\n",
    "bad_value_inf.tns": b"1 1 1 inf\n",
    "bad_value_range.tns": b"1 1 1 1e999\n",
    "bad_value_hex.tns": b"1 1 1 0x10\n",
    "bad_value_text.tns": b"1 1 1 abc\n",
    "value_forms.tns": b"1 1 1 5.\n1 1 2 -.5e1\n1 2 1 1E-300\n2 1 1 123456789012345678901234567890\n2 2 2 1e-320\n",
    "empty.tns": b"# nothing\n\n",
    "duplicate.tns": b"1 1 1 1\n2 2 2 2\n1 1 1 3\n",
    "duplicate_late.tns": b"1 1 1 1\n2 2 2 2\n3 3 3 3\n2 2 2 4\n3 3 3 5\n",
    "order2.tns": b"5 7 1\n1 1 -1\n",
}
# (file, order, skip_header, zero_replace, zero_repl, override)
LOAD_CASES = [
    ("basic.tns", 3, 0, 0, 0.5, []),
    ("basic.tns", 4, 0, 0, 0.5, []),
    ("basic.tns", 1, 0, 0, 0.5, []),
    ("separators.tns", 3, 0, 0, 0.5, []),
    ("header.csv", 3, 1, 0, 0.5, []),
    ("header.csv", 3, 0, 0, 0.5, []),
    ("header_only.csv", 3, 1, 0, 0.5, []),
    ("zero.tns", 3, 0, 0, 0.5, []),
    ("zero.tns", 3, 0, 1, 0.5, []),
    ("zero.tns", 3, 0, 1, -2.0, []),
    ("override.tns", 3, 0, 0, 0.5, [5, 6, 7]),
    ("override.tns", 3, 0, 0, 0.5, [2, 1, 9]),
    ("override.tns", 3, 0, 0, 0.5, [5, 6]),
    ("bad_fields.tns", 3, 0, 0, 0.5, []),
    ("bad_fields_extra.tns", 3, 0, 0, 0.5, []),
    ("bad_index_zero.tns", 3, 0, 0, 0.5, []),
    ("bad_index_alpha.tns", 3, 0, 0, 0.5, []),
    ("bad_index_frac.tns", 3, 0, 0, 0.5, []),
    ("bad_index_plus.tns", 3, 0, 0, 0.5, []),
    ("bad_index_overflow.tns", 3, 0, 0, 0.5, []),
    ("bad_index_neg.tns", 3, 0, 0, 0.5, []),
    ("bad_value_nan.tns", 3, 0, 0, 0.5, []),
    ("bad_value_inf.tns", 3, 0, 0, 0.5, []),
    ("bad_value_range.tns", 3, 0, 0, 0.5, []),
    ("bad_value_hex.tns", 3, 0, 0, 0.5, []),
    ("bad_value_text.tns", 3, 0, 0, 0.5, []),
    ("value_forms.tns", 3, 0, 0, 0.5, []),
    ("empty.tns", 3, 0, 0, 0.5, []),
    ("duplicate.tns", 3, 0, 0, 0.5, []),
    ("duplicate_late.tns", 3, 0, 0, 0.5, []),
    ("order2.tns", 2, 0, 0, 0.5, []),
    ("missing.tns", 3, 0, 0, 0.5, []),
]


def gen_load(L, lines):
    for name, data in LOAD_INPUTS.items():
        with open(name, "wb") as f:
            f.write(data)
    # a multi-chunk file for the threaded reader (the replay sets
    # SPTUCKER_LOAD_CHUNK_BYTES small), with an error deep inside a later chunk
    rng = np.random.default_rng(5)
    n = 2_000
    c = np.stack([rng.permutation(n) + 1, rng.integers(1, 50, n), rng.integers(1, 7, n)], 1)
    v = rng.normal(size=n)
    rows = [f"{a} {b} {d} {x!r}" for (a, b, d), x in zip(c.tolist(), v.tolist())]
    big = "\n".join(rows) + "\n"
    with open("big.tns", "w") as f:
        f.write("# big\n" + big)
    rows[1_337] = "1 2 3"
    with open("big_bad.tns", "w") as f:
        f.write("# big, one short line\n" + "\n".join(rows) + "\n")
    cases = LOAD_CASES + [("big.tns", 3, 0, 0, 0.5, []), ("big_bad.tns", 3, 0, 0, 0.5, [])]
    for k, (name, order, skip, zrep, zval, ovr) in enumerate(cases):
        rc = C.c_int()
        h = L.ref_tensor_load_delimited(name.encode(), order, skip, zrep, zval, len(ovr),
                                        np.array(ovr or [0], np.uint32), C.byref(rc))
        dims, saved, m = "-", "-", ""
        if rc.value == 0:
            d = np.zeros(64, np.uint32)
            nnz = C.c_size_t()
            assert L.ref_tensor_get(h, d, C.byref(nnz), None, None) == 0
            dims = joined(d[:order])
            saved = f"saved_{k:02d}.tns"
            assert L.ref_tensor_save_delimited(h, saved.encode()) == 0, msg(L)
            O.ref().ref_tensor_free(h)
        else:
            m = msg(L)
        lines.append(["load", name, order, skip, zrep, repr(float(zval)), joined(ovr), rc.value, dims, saved, m])


def gen_model(L, lines):
    dims, J, R = [7, 5, 4], [3, 3, 2], 2
    m = O.RefModel(np.array(dims, np.uint32), J, R).init_gaussian(0.5, 0.1, 11)
    assert L.ref_model_save(m.h, b"model_ref.bin") == 0
    lines.append(["modelgen", joined(dims), joined(J), R, repr(0.5), repr(0.1), 11, "model_ref.bin"])
    good = open("model_ref.bin", "rb").read()
    hdr = 8 + 4 + 4 + 8 * 3 + 8 * 3 + 8  # magic, version, order, dims, J, R

    def put(off, fmt, val, src=good):
        b = bytearray(src)
        struct.pack_into(fmt, b, off, val)
        return bytes(b)

    bad = {
        "model_truncated.bin": good[:-3],
        "model_header_only.bin": good[:20],
        "model_magic.bin": b"SPTUCKX\0" + good[8:],
        "model_version.bin": put(8, "<I", 2),
        "model_order.bin": put(12, "<I", 1),
        "model_dim0.bin": put(16 + 8, "<Q", 0),
        "model_dimbig.bin": put(16, "<Q", 1 << 33),
        "model_rank0.bin": put(16 + 24 + 8, "<Q", 0),
        "model_rcore0.bin": put(16 + 48, "<Q", 0),
        "model_rcore_gt_j.bin": put(16 + 48, "<Q", 3),
        "model_trailing.bin": good + b"\0",
        "model_nan.bin": put(hdr + 8 * 5, "<d", float("nan")),
        "model_empty.bin": b"",
    }
    for name, data in bad.items():
        with open(name, "wb") as f:
            f.write(data)
    for name in ["model_ref.bin", *bad, "model_missing.bin"]:
        rc, order, R_ = C.c_int(), C.c_int(), C.c_uint32()
        d, j = np.zeros(64, np.uint32), np.zeros(64, np.uint32)
        h = L.ref_model_load(name.encode(), C.byref(order), d, j, C.byref(R_), C.byref(rc))
        resaved, m = "-", ""
        if rc.value == 0:
            resaved = "resaved_" + name
            assert L.ref_model_save(h, resaved.encode()) == 0
            O.ref().ref_model_free(h)
        else:
            m = msg(L)
        lines.append(["model", name, rc.value, resaved, m])


def gen_metrics(L, lines):
    nan = float("nan")
    rows = np.array([
        [0, 0.125, 1.5, 1.625, 0.9, 0.7, nan, nan, 123456, 240],
        [1, 1e-9, 2.0 / 3.0, 2.0 / 3.0 + 1e-9, 0.5, 0.25, 0.75, 0.6, 0, 240],
        [17, 3.5e-310, 1e300, 1e300, 1.0, 1.0, 1.0, 1.0, 2 ** 52, 2 ** 40],
    ], np.float64)
    comments = ["config: J=10 R=10", "", "seed 1 # nested hash"]
    assert L.ref_write_metrics_csv(b"metrics_ref.csv", len(rows), np.ascontiguousarray(rows),
                                   "\n".join(comments).encode() + b"\n") == 0, msg(L)
    lines.append(["mwrite", "metrics_ref.csv", "|".join(comments),
                  ";".join(",".join(float(x).hex() for x in r) for r in rows)])
    bad = {
        "metrics_header.csv": b"epoch,core_s\n0,1\n",
        "metrics_fields.csv": open("metrics_ref.csv", "rb").read() + b"3,1,2\n",
        "metrics_num.csv": open("metrics_ref.csv", "rb").read() + b"3,x,1,1,1,1,1,1,1,1\n",
        "metrics_int.csv": open("metrics_ref.csv", "rb").read() + b"3,1,1,1,1,1,1,1,-5,1\n",
        "metrics_noheader.csv": b"# only comments\n\n",
        "metrics_crlf.csv": open("metrics_ref.csv", "rb").read().replace(b"\n", b"\r\n"),
    }
    for name, data in bad.items():
        with open(name, "wb") as f:
            f.write(data)
    for name in ["metrics_ref.csv", *bad, "metrics_missing.csv"]:
        out = np.zeros(64 * 10)
        n = C.c_size_t()
        com = C.create_string_buffer(4096)
        rc = L.ref_parse_metrics_csv(name.encode(), 64, out, C.byref(n), com, 4096)
        cm = com.value.decode().rstrip("\n").split("\n") if rc == 0 and com.value else []
        lines.append(["mparse", name, rc, n.value if rc == 0 else 0, "|".join(cm) if cm else "-",
                      msg(L) if rc else ""])


def gen_synth(L, lines):
    for dims, tJ, tR, nnz, noise, tmean, tsd, seed in [
        ([9, 8, 7, 6], [3, 2, 2, 2], 2, 300, 0.05, 0.5, 0.1, 3),    # pool path (total <= 2^22)
        ([3000, 2000, 1000], [3, 3, 3], 2, 500, 0.0, 0.0, 1.0, 9),  # rejection path
    ]:
        d = np.array(dims, np.uint32)
        c = np.empty(nnz * len(dims), np.uint32)
        v = np.empty(nnz)
        assert O.ref().ref_synth_planted(len(dims), d, np.array(tJ, np.uint32), tR, nnz, noise, tmean, tsd,
                                         seed, c, v) == 0
        t = O.RefTensor(d, c, v)
        name = f"planted_{seed}.tns"
        assert L.ref_tensor_save_delimited(t.h, name.encode()) == 0
        lines.append(["planted", joined(dims), joined(tJ), tR, nnz, repr(noise), repr(tmean), repr(tsd), seed,
                      name])
    for dims, tJ, tR, nnz, seed, tm, ts, noise, half, lo, hi in [
        ([40, 30, 20], [3, 3, 3], 3, 900, 4, 3.0, 0.9, 0.4, 1, 0.5, 5.0),
        ([40, 30, 20], [3, 3, 3], 3, 900, 4, 3.0, 1.0, 0.0, 0, 1.0, 5.0),
        ([50, 40, 30, 20], [2, 2, 2, 2], 2, 700, 8, 0.0, 2.0, 0.1, 1, -3.0, 3.0),
    ]:
        d = np.array(dims, np.uint32)
        c = np.empty(nnz * len(dims), np.uint32)
        v = np.empty(nnz)
        assert L.ref_synth_ratings(len(dims), d, np.array(tJ, np.uint32), tR, nnz, 0.5, 0.1, seed, tm, ts, noise,
                                   half, lo, hi, c, v) == 0, msg(L)
        t = O.RefTensor(d, c, v)
        name = f"ratings_{seed}_{half}.tns"
        assert L.ref_tensor_save_delimited(t.h, name.encode()) == 0
        lines.append(["ratings", joined(dims), joined(tJ), tR, nnz, repr(0.5), repr(0.1), seed, repr(tm), repr(ts),
                      repr(noise), half, repr(lo), repr(hi), name])


def gen_index(L, lines):
    cases = [
        ([4, 3, 2], [1, 1, 1], 0), ([4, 3, 2], [4, 3, 2], 0), ([4, 3, 2], [2, 3, 1], 1),
        ([4, 3, 2], [3, 2, 2], 2), ([5, 7, 3, 2], [5, 1, 3, 2], 3), ([100000, 90000, 80000], [99999, 1, 77777], 1),
        ([4, 3, 2], [5, 1, 1], 0), ([4, 3, 2], [0, 1, 1], 1), ([4, 3, 2], [1, 1, 1], 3),
    ]
    for dims, coord, mode in cases:
        col, vec = C.c_uint64(), C.c_uint64()
        inv = np.zeros(len(dims), np.uint32)
        rc = L.ref_indexing(len(dims), np.array(dims, np.uint32), np.array(coord, np.uint32), mode, C.byref(col),
                            C.byref(vec), inv)
        lines.append(["index", joined(dims), joined(coord), mode, rc, col.value if rc == 0 else 0,
                      vec.value if rc == 0 else 0, joined(inv) if rc == 0 else "-", msg(L) if rc else ""])


def generate(out_dir: str) -> None:
    L = lib()
    if os.path.isdir(out_dir):
        shutil.rmtree(out_dir)
    os.makedirs(out_dir)
    cwd = os.getcwd()
    os.chdir(out_dir)
    try:
        lines: list[list] = []
        gen_load(L, lines)
        gen_model(L, lines)
        gen_metrics(L, lines)
        gen_synth(L, lines)
        gen_index(L, lines)
        with open("cases.txt", "w") as f:
            for ln in lines:
                f.write("\t".join(str(x) for x in ln) + "\n")
    finally:
        os.chdir(cwd)


if __name__ == "__main__":
    O.build_oracle(ref=True)
    generate(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "io"))
    print("wrote tests/golden/io")
