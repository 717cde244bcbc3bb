"""Op-trace files: the reference's text format
(trace_format.cpp:34-126) and the packed binary form with its streaming chunk
reader. Host-only, so these run without a GPU; the replay test is gpu."""
import numpy as np
import pytest


@pytest.fixture()
def tio():
    from paper_1908_09378_b200 import trace_io
    return trace_io


def test_text_round_trip(tio, O, tmp_path):
    tr = O.gen_legal_trace(3000, 8, 5)
    p = tmp_path / "t.txt"
    tio.save_text(tr, p)
    back = tio.load_text(p)
    assert back.n_ops == tr.n_ops
    assert np.array_equal(back.kinds, tr.kinds)
    assert np.array_equal(back.offsets, tr.offsets)
    assert np.array_equal(back.vals, tr.vals)
    keep = np.repeat(tr.kinds, np.diff(tr.offsets).astype(np.int64)) != ord("D")
    assert np.array_equal(back.prios[keep], np.asarray(tr.prios)[keep])


def test_text_format_lines(tio, tmp_path):
    p = tmp_path / "t.txt"
    p.write_text("# a comment\n\nU 3 10\nB 2 1 5 4 6   # trailing comment\nE\nD 3\n")
    t = tio.load_text(p)
    assert bytes(t.kinds) == b"UBED"
    assert t.offsets.tolist() == [0, 1, 3, 3, 4]
    assert t.vals.tolist() == [3, 1, 4, 3]
    assert t.prios.tolist()[:3] == [10, 5, 6]
    assert p.read_text().count("\n") == 6


@pytest.mark.parametrize("body,op,what", [
    ("U 1 2\nX 5\n", 1, "unknown op 'X'"),
    ("U 1 2\nE\nB 0\n", 2, "empty batch"),
    ("E extra\n", 0, "trailing tokens"),
    ("U 1\n", 0, "missing or bad priority"),
    ("U 4294967296 1\n", 0, "value out of range"),
    ("UU 1 2\n", 0, "unknown op 'UU'"),
])
def test_text_errors_carry_op_and_line(tio, tmp_path, body, op, what):
    from paper_1908_09378_b200 import TraceError
    p = tmp_path / "bad.txt"
    p.write_text(body)
    with pytest.raises(TraceError) as ei:
        tio.load_text(p)
    assert ei.value.op_index == op
    assert what in str(ei.value)
    assert "line" in str(ei.value)


def test_missing_file(tio, tmp_path):
    from paper_1908_09378_b200 import TraceError
    with pytest.raises(TraceError):
        tio.load_text(tmp_path / "nope.txt")
    with pytest.raises(TraceError):
        tio.BinaryTraceReader(tmp_path / "nope.pbht")


def test_binary_round_trip_and_chunks(tio, O, tmp_path):
    tr = O.gen_legal_trace(5000, 64, 9)
    p = tmp_path / "t.pbht"
    tio.save_binary(tr, p)
    with tio.BinaryTraceReader(p) as r:
        assert r.n_ops == tr.n_ops and r.n_elems == len(tr.vals)
        whole = r.read(0, r.n_ops)
        assert np.array_equal(whole.kinds, tr.kinds)
        assert np.array_equal(whole.offsets, tr.offsets)
        assert np.array_equal(whole.vals, tr.vals)
        assert np.array_equal(whole.prios, tr.prios)
        got_k, got_v = [], []
        for op0, ch in r.chunks(777):
            assert ch.offsets[0] == 0
            got_k.append(ch.kinds)
            got_v.append(ch.vals)
            b, e = int(tr.offsets[op0]), int(tr.offsets[op0 + ch.n_ops])
            assert np.array_equal(ch.prios, tr.prios[b:e])
        assert np.array_equal(np.concatenate(got_k), tr.kinds)
        assert np.array_equal(np.concatenate(got_v), tr.vals)


def test_binary_rejects_garbage(tio, tmp_path):
    from paper_1908_09378_b200 import TraceError
    p = tmp_path / "g.pbht"
    p.write_bytes(b"not a trace at all, definitely")
    with pytest.raises(TraceError):
        tio.BinaryTraceReader(p)


def test_text_and_binary_agree(tio, O, tmp_path):
    tr = O.gen_mixed_trace(400, 1 << 12, 64, 3)
    tio.save_text(tr, tmp_path / "a.txt")
    tio.save_binary(tio.load_text(tmp_path / "a.txt"), tmp_path / "a.pbht")
    with tio.BinaryTraceReader(tmp_path / "a.pbht") as r:
        b = r.read(0, r.n_ops)
    assert np.array_equal(b.kinds, tr.kinds) and np.array_equal(b.vals, tr.vals)
    assert np.array_equal(b.prios, tr.prios)


@pytest.mark.gpu
def test_chunked_replay_matches_oracle(pbh, tio, O, tmp_path):
    tr = O.gen_legal_trace(20000, 64, 13)
    p = tmp_path / "r.pbht"
    tio.save_binary(tr, p)
    want_v, want_p = O.run_oracle(tr)
    eng = pbh.Engine(pbh.EngineConfig(d=64, debug_assertions=True))
    v, pr, ms = tio.run_trace_file(eng, p, chunk_ops=1500)
    assert np.array_equal(v, want_v) and np.array_equal(pr, want_p)
    assert eng.check_invariants() == []


_TRICKY = [
    "U 1 2\n", "U\t1\t2\r\n", "  U   7 8   \n", "B 2 1 5 4 6\n", "B 1 3 +9\n", "U +4 5\n",
    "U 1 -1\n", "U -1 3\n", "U 1 18446744073709551615\n", "U 1 18446744073709551616\n",
    "U 4294967295 0\n", "U 4294967296 0\n", "U 1 2x\n", "U 1x 2\n", "U 1 2 # c\n",
    "U 1 2#c\n", "U 1# 2\n", "#only\n\n\n", "", "E\nE\n", "E x\n", "D 5\n", "D\n",
    "D 5 6\n", "B 0\n", "B 16777217 1 1\n", "B 2 1 2\n", "B 2 1 2 3\n", "B x\n",
    "X\n", "UU 1 2\n", "u 1 2\n", "U 1 2\nE\nD 1\nB 3 1 1 2 2 3 3\nE\n", "U 1 2", "\n\nE",
    "U 00012 0003\n", "U 1\x0b2\n", "U 1\x0c2\n", "U - 2\n", "U + 2\n", "U 1 --2\n",
]


@pytest.mark.skipif(not __import__("os").path.exists(__import__("os").path.join(
    __import__("os").path.dirname(__file__), "..", "oracle", "_ref", "libpbhref.so")),
    reason="oracle/_ref not built")
@pytest.mark.parametrize("i", range(len(_TRICKY)))
def test_text_parser_matches_reference(tio, O, tmp_path, i):
    """Our single-pass tokenizer against the reference's istream parser
    (trace_format.cpp:34-98) on edge cases: same ops, or same op index and
    message."""
    from paper_1908_09378_b200 import TraceError
    p = tmp_path / "t.txt"
    p.write_bytes(_TRICKY[i].encode())
    try:
        want = O.ref_load_text(p)
        werr = None
    except O.RefError as e:
        want, werr = None, e
    try:
        got = tio.load_text(p)
        gerr = None
    except TraceError as e:
        got, gerr = None, e
    if werr is not None:
        assert gerr is not None, f"reference rejects {_TRICKY[i]!r}: {werr}"
        assert gerr.op_index == werr.op_index
        assert str(werr).split(": ", 1)[1] in str(gerr)
    else:
        assert gerr is None, f"reference accepts {_TRICKY[i]!r}: {gerr}"
        assert np.array_equal(got.kinds, want.kinds)
        assert np.array_equal(got.offsets, want.offsets)
        assert np.array_equal(got.vals, want.vals)
        keep = np.repeat(want.kinds, np.diff(want.offsets).astype(np.int64)) != ord("D")
        assert np.array_equal(np.asarray(got.prios)[keep], np.asarray(want.prios)[keep])
