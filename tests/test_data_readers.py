"""Real-data readers: LIBSVM -> CSR and IDX -> dense, the inputs of the device
shards. The product readers (csrc/data_io.cu, host code behind the C ABI) are checked bit-for-bit
against the reference's own load_libsvm / load_idx (src/data_io.cpp:85-137, 220-271) built in
oracle/_ref: same arrays, or the same error class and message, on hand-written edge cases and on
seeded random files. The GPU test feeds a loaded file through a device shard."""
import struct

import numpy as np
import pytest

import paper_1807_07132_b200 as nadmm
from oracle import OracleError

_CODE = {nadmm.ConfigError: 2, nadmm.DataError: 12}


def _both(ref, load_ours, load_ref):
    try:
        ours = load_ours()
        err = None
    except (nadmm.ConfigError, nadmm.DataError) as e:
        ours, err = None, e
    try:
        theirs = load_ref()
        rerr = None
    except OracleError as e:
        theirs, rerr = None, e
    if rerr is not None or err is not None:
        assert err is not None and rerr is not None, (err, rerr)
        assert rerr.code == _CODE[type(err)], (err, rerr)
        assert str(rerr) == f"[{rerr.code}] {err}"
        return None
    assert (ours.n, ours.p, ours.num_classes) == (theirs["n"], theirs["p"], theirs["C"])
    assert np.array_equal(ours.labels, theirs["labels"])
    assert np.array_equal(ours.label_values, theirs["label_values"])
    if ours.sparse:
        assert np.array_equal(ours.indptr, theirs["indptr"])
        assert np.array_equal(ours.indices, theirs["indices"])
        assert ours.vals.tobytes() == theirs["vals"].tobytes()
    else:
        assert ours.X.tobytes() == theirs["X"].tobytes()
    return ours


def _libsvm(ref, path, text):
    path.write_bytes(text.encode() if isinstance(text, str) else text)
    return _both(ref, lambda: nadmm.read_libsvm(path), lambda: ref.load_libsvm(path))


LIBSVM_OK = [
    "# header comment\n3 2:1.5 1:2 2:0.5\n-1 5:1e-3\n\n3 1:0\n7\n",  # comments, blanks, dups, empty rows
    "+2 1:1\n1 1:2\n",                    # signed label
    "1e0 1:1\n2.0 3:4\n5. 2:1\n",         # exponent / trailing-dot integer labels
    "1 1:2abc\n2 3x:1\n",                 # stoll/stod accept partial parses
    "1\t1:2\r\n2 1:1\r\n",                # tabs and CRLF
    "1 1:1 1:2 1:-3\n2 2:1\n",            # duplicates summed to exact 0
    "1 4:1 2:2 3:3 1:4\n2 1:1\n",         # unsorted columns
    "1 1:1e-310\n2 1:1\n",                # subnormal value (strtod range rules)
    "0 1:1\n-0 1:2\n1 2:1\n",             # -0 and 0 are one label
    "1 1:0x10\n2 1:1\n",                  # hex value through strtod
    "1 1:inf\n2 1:1\n",                   # non-finite value -> Dataset validation
    "1 1:nan\n2 1:1\n",
]

LIBSVM_BAD = [
    "1.5 1:2\n2 1:1\n",                   # non-integer label
    "abc 1:2\n",
    "inf 1:1\n2 1:1\n",                   # istream does not read inf
    "1e 1:1\n2 1:1\n",                    # incomplete exponent
    ".\n",
    "   \n",                              # whitespace-only line is not blank
    "0x1 1:1\n2 1:1\n",                   # label 0, then token 'x1'
    "1 2\n",                              # no colon
    "1 a:2\n",
    "1 2:x\n",
    "1 :5\n",
    "1 1:\n",
    "1 0:1\n",                            # 0-based index
    "1 -3:1\n",
    "1 1:1e400\n2 1:1\n",                 # stod out_of_range
    "1 99999999999999999999:1\n",         # stoll out_of_range
    "1:2 3:4\n",                          # label glued to a token
    "# only comments\n\n",                # no data rows
    "",
    "3 1:1\n3 2:1\n",                     # one class
    "1\n2\n",                             # p = 0
]


@pytest.mark.parametrize("text", LIBSVM_OK)
def test_libsvm_matches_reference(ref, tmp_path, text):
    _libsvm(ref, tmp_path / "d.svm", text)


@pytest.mark.parametrize("text", LIBSVM_BAD)
def test_libsvm_errors_match_reference(ref, tmp_path, text):
    path = tmp_path / "d.svm"
    path.write_text(text)
    with pytest.raises((nadmm.ConfigError, nadmm.DataError)):
        nadmm.read_libsvm(path)
    _libsvm(ref, path, text)


def test_libsvm_missing_file(ref, tmp_path):
    with pytest.raises(nadmm.ConfigError, match="cannot open"):
        nadmm.read_libsvm(tmp_path / "absent.svm")
    _both(ref, lambda: nadmm.read_libsvm(tmp_path / "absent.svm"), lambda: ref.load_libsvm(tmp_path / "absent.svm"))


def _random_libsvm(rng, rows, bad_rate):
    vocab_bad = ["x", "1:", ":2", "0:1", "a:b", "1.5", "2:1e999"]
    lines = []
    for _ in range(rows):
        r = rng.random()
        if r < 0.05:
            lines.append("# comment")
            continue
        if r < 0.08:
            lines.append("")
            continue
        toks = [str(int(rng.integers(-3, 6)))]
        for _ in range(int(rng.integers(0, 12))):
            if rng.random() < bad_rate:
                toks.append(vocab_bad[int(rng.integers(len(vocab_bad)))])
            else:
                v = rng.normal() * 10 ** float(rng.integers(-8, 8))
                fmt = ["{:.17g}", "{:.3f}", "{:e}", "{!r}"][int(rng.integers(4))]
                toks.append(f"{int(rng.integers(1, 300))}:{fmt.format(v)}")
        lines.append(rng.choice([" ", "\t", "  "]).join(toks))
    return "\n".join(lines) + ("\n" if rng.random() < 0.5 else "")


@pytest.mark.parametrize("seed", range(24))
def test_libsvm_fuzz_matches_reference(ref, tmp_path, seed):
    rng = np.random.default_rng(seed)
    text = _random_libsvm(rng, int(rng.integers(1, 400)), 0.0 if seed % 3 else 0.01)
    _libsvm(ref, tmp_path / "f.svm", text)


def _idx_files(tmp_path, n, rows, cols, labels, pixels=None, img_magic=0x803, lab_magic=0x801, n_labels=None,
               cut_img=0, cut_lab=0):
    rng = np.random.default_rng(n * 31 + rows)
    if pixels is None:
        pixels = rng.integers(0, 256, size=n * rows * cols, dtype=np.uint8)
    img = struct.pack(">IIII", img_magic, n, rows, cols) + bytes(pixels)
    lab = struct.pack(">II", lab_magic, n if n_labels is None else n_labels) + bytes(np.asarray(labels, np.uint8))
    fi, fl = tmp_path / "img.idx", tmp_path / "lab.idx"
    fi.write_bytes(img[:len(img) - cut_img])
    fl.write_bytes(lab[:len(lab) - cut_lab])
    return fi, fl


def _idx(ref, fi, fl):
    return _both(ref, lambda: nadmm.read_idx(fi, fl), lambda: ref.load_idx(fi, fl))


def test_idx_matches_reference(ref, tmp_path):
    rng = np.random.default_rng(5)
    fi, fl = _idx_files(tmp_path, 97, 7, 5, rng.integers(0, 10, 97))
    d = _idx(ref, fi, fl)
    assert d is not None and d.X.shape == (97, 35) and d.X.max() <= 1.0


def test_idx_full_byte_range(ref, tmp_path):
    fi, fl = _idx_files(tmp_path, 256, 1, 1, np.arange(256) % 4, pixels=np.arange(256, dtype=np.uint8))
    d = _idx(ref, fi, fl)
    assert d.num_classes == 4 and np.array_equal(d.label_values, [0, 1, 2, 3])


@pytest.mark.parametrize("case", ["img_magic", "lab_magic", "count", "cut_img", "cut_lab", "header", "one_class",
                                  "no_rows", "no_pixels"])
def test_idx_errors_match_reference(ref, tmp_path, case):
    kw = dict(n=6, rows=2, cols=3, labels=[0, 1, 2, 1, 0, 3])
    if case == "img_magic":
        kw["img_magic"] = 0x802
    elif case == "lab_magic":
        kw["lab_magic"] = 0x803
    elif case == "count":
        kw["n_labels"] = 5
    elif case == "cut_img":
        kw["cut_img"] = 4
    elif case == "cut_lab":
        kw["cut_lab"] = 1
    elif case == "header":
        kw["cut_img"] = 36 + 6
    elif case == "one_class":
        kw["labels"] = [0] * 6  # C = max digit + 1 = 1
    elif case == "no_rows":
        kw.update(n=0, labels=[])
    elif case == "no_pixels":
        kw.update(rows=0)
    fi, fl = _idx_files(tmp_path, **kw)
    with pytest.raises((nadmm.ConfigError, nadmm.DataError)):
        nadmm.read_idx(fi, fl)
    _idx(ref, fi, fl)


def test_idx_missing_file(tmp_path):
    with pytest.raises(nadmm.ConfigError, match="cannot open"):
        nadmm.read_idx(tmp_path / "a", tmp_path / "b")


@pytest.mark.gpu
def test_loaded_libsvm_shard_matches_reference(ref, tmp_path):
    """A LIBSVM file through load_libsvm -> device shard gives the reference's Hv on its own load."""
    from oracle import Shard

    rng = np.random.default_rng(11)
    path = tmp_path / "s.svm"
    path.write_text(_random_libsvm(rng, 700, 0.0))
    ds = nadmm.load_libsvm(path)
    r = ref.load_libsvm(path)
    assert np.array_equal(ds.label_values(), r["label_values"])
    rd = ref.dataset(Shard(labels=r["labels"], C_=r["C"], csr=(r["indptr"], r["indices"], r["vals"]), p=r["p"]))
    d = ds.weight_dim()
    w, v = rng.normal(size=d) * 0.01, rng.normal(size=d)
    hv = nadmm.hessian_vec(ds, w, v, 1e-3)
    hr = rd.hessian_vec(w, v, 1e-3)
    assert np.max(np.abs(hv - hr)) <= 1e-12 * max(1.0, np.max(np.abs(hr)))
    assert nadmm.loss(ds, w, 1e-3) == pytest.approx(rd.loss(w, 1e-3), rel=1e-12)
