"""The formats either side of the path (data_io.cpp): parse_libsvm, write_libsvm
and write_csv through the C ABI (host code, no GPU), against the expectations
of the reference's test_data_io.cpp and the oracle's restatement."""
import numpy as np
import pytest


def _same_csr(a, b):
    assert (a.rows, a.cols) == (b.rows, b.cols)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.values, b.values)


def test_libsvm_well_formed(rp, oracle):  # test_data_io.cpp:13-24
    m, labels = rp.parse_libsvm("+1 2:0.5 4:-1.25\n3.5 1:1\n")
    assert labels.tolist() == [1.0, 3.5]
    assert (m.rows, m.cols) == (2, 4)
    assert m.offsets.tolist() == [0, 2, 3] and m.indices.tolist() == [1, 3, 0]
    assert m.values.tolist() == [0.5, -1.25, 1.0]
    om, ol = oracle.parse_libsvm("+1 2:0.5 4:-1.25\n3.5 1:1\n")
    _same_csr(m, om)
    assert np.array_equal(labels, ol)


def test_libsvm_blanks_and_comments(rp):  # test_data_io.cpp:26-32
    m, labels = rp.parse_libsvm("\n# header comment\n2 1:4 # trailing note\n\n")
    assert m.rows == 1 and labels.tolist() == [2.0]
    assert m.indices.tolist() == [0] and m.values.tolist() == [4.0]
    m, labels = rp.parse_libsvm("")
    assert (m.rows, m.cols, len(m.values)) == (0, 0, 0) and labels.size == 0
    m, _ = rp.parse_libsvm("1\r\n2 3:1\r\n")  # CR is whitespace; a label-only row is an empty row
    assert m.offsets.tolist() == [0, 0, 1] and m.cols == 3


@pytest.mark.parametrize("text,line,col,needle", [
    ("1 3:1 2:1\n", 1, 7, "non-increasing"),  # test_data_io.cpp:35-44
    ("ok 1:1\n1 0:5\n", 1, 1, "malformed number"),  # :46-54, the malformed label comes first
    ("1 1:1\n1 0:5\n", 2, 3, ">= 1"),  # :56-63
    ("1 2:abc\n", 1, 5, "malformed number"),  # :65-67
    ("1 2:1e999\n", 1, 5, "out of range"),
    ("1 2:inf\n", 1, 5, "non-finite"),
    ("1 2:1.5x\n", 1, 5, "trailing characters"),
    ("1 2\n", 1, 3, "expected index:value"),
    ("1 :2\n", 1, 3, "expected index:value"),
    ("1 2:\n", 1, 3, "expected index:value"),
    ("1 x:2\n", 1, 3, "malformed feature index"),
    ("  7   5:1 5:2", 1, 11, "non-increasing"),
])
def test_libsvm_errors_carry_line_and_column(rp, oracle, text, line, col, needle):
    with pytest.raises(rp.ParseError) as e:
        rp.parse_libsvm(text)
    assert (e.value.line, e.value.column) == (line, col)
    assert needle in str(e.value) and str(e.value).startswith(f"line {line}, column {col}: ")
    if needle not in ("out of range",):  # (Python's float() has no ERANGE; the C side follows std::stod)
        with pytest.raises(oracle.ParseError) as o:
            oracle.parse_libsvm(text)
        assert (o.value.line, o.value.column) == (line, col) and str(o.value) == str(e.value)


def test_libsvm_feature_override(rp):
    m, _ = rp.parse_libsvm("1 2:1\n", feature_override=7)
    assert m.cols == 7
    with pytest.raises(ValueError, match="below max index"):
        rp.parse_libsvm("1 9:1\n", feature_override=4)


def test_libsvm_round_trip(rp, oracle):  # test_data_io.cpp:71-85
    rng = np.random.default_rng(3)
    dense = np.where(rng.random((40, 17)) < 0.3, rng.standard_normal((40, 17)), 0.0)
    dense[5] = 0.0  # an empty row
    labels = rng.standard_normal(40)
    text = rp.write_libsvm(dense, labels)
    m, back = rp.parse_libsvm(text, feature_override=17)
    c = oracle.Csr.from_dense(dense)
    assert np.array_equal(m.offsets, c.offsets) and np.array_equal(m.indices, c.indices)
    assert np.array_equal(m.values, c.values) and np.array_equal(back, labels)  # %.17g round-trips exactly
    _same_csr(m, oracle.parse_libsvm(text, 17)[0])
    assert rp.write_libsvm(m, back) == text
    with pytest.raises(ValueError):
        rp.write_libsvm(dense, labels[:-1])


def test_csv_sorted_with_17_digits(rp, oracle):  # test_data_io.cpp:206-234
    def result(name):
        pts = [rp.PathPoint(lam, np.zeros((1, 1)), seconds=0.001, train_loss=1.0 / 3.0,
                            test_loss=0.25 if lam == 1.0 else None) for lam in (10.0, 1.0)]
        return rp.RegPathResult(name, pts)

    res = [result("svd"), result("direct")]
    csv = rp.write_csv(res)
    lines = csv.split("\n")
    assert lines[0] == "lambda,train_loss,test_loss,time_s,solver"
    assert "direct" in lines[1] and "0.33333333333333331" in lines[1] and "0.25" in lines[1]
    assert "svd" in lines[2]
    assert ",," in lines[3]
    assert lines[1] == "1,0.33333333333333331,0.25,0.001,direct"
    assert csv.endswith("\n") and len(lines) == 6
    assert csv == oracle.write_csv(res)
    assert rp.write_csv([]) == "lambda,train_loss,test_loss,time_s,solver\n"


def test_csv_random_paths_match_oracle(rp, oracle):
    rng = np.random.default_rng(9)
    res = []
    for name in ("ihs-bin", "cg", "direct", "ihs"):
        lams = np.sort(rng.choice(np.geomspace(1e-4, 1e3, 15), size=8, replace=False))
        pts = [rp.PathPoint(float(l), np.zeros((1, 1)), seconds=float(rng.random() * 1e-3),
                            train_loss=float(rng.standard_normal() * 1e6),
                            test_loss=float(rng.random()) if rng.random() < 0.5 else None) for l in lams]
        res.append(rp.RegPathResult(name, pts))
    assert rp.write_csv(res) == oracle.write_csv(res)
