"""Triplet text I/O (dfcg_load_triplets_* / dfcg_save_triplets_file, include/dfcg_host.h) against
the reference's own loader tests (P/tests/test_matrix_io.cpp:24-122) and a line-by-line Python
restatement of load_triplets (P/include/dfc/matrix_io.hpp:125-170) on ragged inputs. CPU only."""
import os

import numpy as np
import pytest

import paper_1107_0789_b200 as P


def entries(o):
    return list(zip(o.rows.tolist(), o.cols.tolist(), o.vals.tolist()))


def test_header_and_single_entry():  # test_matrix_io.cpp:24-32
    o = P.parse_triplets("% 2 2\n0 0 1.5\n")
    assert (o.m, o.n, o.count) == (2, 2, 1)
    assert entries(o) == [(0, 0, 1.5)]


def test_header_only_gives_empty_matrix():  # :34-39
    o = P.parse_triplets("% 3 4\n")
    assert (o.m, o.n, o.count) == (3, 4, 0)


def test_dims_inferred_without_header():  # :41-46
    o = P.parse_triplets("0 0 1\n4 2 -3.5\n")
    assert (o.m, o.n, o.count) == (5, 3, 2)


def test_one_based():  # :48-54
    o = P.parse_triplets("% 2 2\n1 1 9\n2 2 7\n", one_based=True)
    assert entries(o) == [(0, 0, 9.0), (1, 1, 7.0)]


def test_blank_lines_ignored():  # :56-59
    assert P.parse_triplets("\n% 2 2\n\n0 1 3\n\n").count == 1


def test_duplicate_rejected():  # :61-63
    with pytest.raises(ValueError, match="duplicate entry"):
        P.parse_triplets("% 2 2\n0 0 1\n0 0 2\n")


def test_malformed_line_reports_line_number():  # :65-73
    with pytest.raises(P.ParseError) as e:
        P.parse_triplets("% 2 2\n0 zebra 1\n")
    assert e.value.line == 2 and "line 2" in str(e.value)


def test_trailing_tokens_rejected():  # :75-78
    with pytest.raises(P.ParseError, match="trailing tokens"):
        P.parse_triplets("0 0 1 junk\n")
    with pytest.raises(P.ParseError, match="trailing tokens in header"):
        P.parse_triplets("% 2 2 9\n")


def test_index_outside_declared_dims():  # :80-83
    with pytest.raises(IndexError, match="line 2: index outside declared 2x2"):
        P.parse_triplets("% 2 2\n2 0 1\n")
    with pytest.raises(IndexError):
        P.parse_triplets("% 2 2\n0 5 1\n")


def test_negative_index_rejected():  # :85-88
    with pytest.raises(P.ParseError, match="negative index"):
        P.parse_triplets("-1 0 1\n")
    with pytest.raises(P.ParseError):
        P.parse_triplets("% 2 2\n0 0 1\n", one_based=True)  # one-based 0 underflows


def test_header_after_data_rejected():  # :90-93
    with pytest.raises(P.ParseError, match="unexpected header"):
        P.parse_triplets("0 0 1\n% 2 2\n")
    with pytest.raises(P.ParseError, match="unexpected header"):
        P.parse_triplets("% 2 2\n% 2 2\n")


def test_empty_input_rejected():  # :95-97
    with pytest.raises(ValueError, match="no header and no data"):
        P.parse_triplets("")
    with pytest.raises(ValueError):
        P.parse_triplets("\n  \n")


def test_bad_header_dims():
    for text in ("% 0 2\n", "% 2\n", "% a b\n", "% 2 -1\n"):
        with pytest.raises(P.ParseError, match="bad header dims"):
            P.parse_triplets(text)


def test_values_istream_forms():
    o = P.parse_triplets("0 0 1e3\n1 0 -.5\n2 0 +2.\n3 0 1E-2\r\n")
    assert o.vals.tolist() == [1000.0, -0.5, 2.0, 0.01]
    for bad in ("0 0 inf\n", "0 0 nan\n", "0 0 1e999\n", "0 0\n", "0 0 .\n", "0.5 0 1\n"):
        with pytest.raises(P.ParseError):
            P.parse_triplets(bad)
    with pytest.raises(P.ParseError, match="trailing tokens"):
        P.parse_triplets("0 0 1.5abc\n")


def test_save_round_trip_exact(tmp_path):  # :99-122
    rng = P.SeededRng(17, 0)
    u, z = rng.uniform(64), rng.normal(64)
    rows, cols, vals = [], [], []
    k = 0
    for j in range(7):
        for i in range(5):
            if i == 0 and j == 0:
                continue
            if u[k] < 0.5:
                rows.append(i), cols.append(j), vals.append(z[k] * 1e3)
            k += 1
    rows.insert(0, 0), cols.insert(0, 0), vals.insert(0, 1.0 / 3.0)
    obs = P.Observed(5, 7, np.array(rows), np.array(cols), np.array(vals))
    back = P.parse_triplets(P.format_triplets(obs))
    assert (back.m, back.n) == (5, 7)
    assert entries(back) == entries(obs)  # %.17g is lossless: bit for bit
    path = tmp_path / "obs.txt"
    P.save_triplets(path, obs)
    assert open(path).read() == P.format_triplets(obs)
    assert entries(P.load_triplets(path)) == entries(obs)


def _ref_load(text, one_based=False):
    """Restatement of load_triplets (matrix_io.hpp:127-170) + the ObservedMatrix ctor order."""
    base = 1 if one_based else 0
    m = n = -1
    obs, seen = [], False
    for lineno, line in enumerate(text.split("\n"), 1):
        tok = line.split()
        if not tok:
            continue
        if tok[0] == "%":
            assert not seen and m < 0
            m, n = int(tok[1]), int(tok[2])
            continue
        i, j, v = int(tok[0]) - base, int(tok[1]) - base, float(tok[2])
        seen = True
        obs.append((j, i, v))
    if m < 0:
        m = max(o[1] for o in obs) + 1
        n = max(o[0] for o in obs) + 1
    obs.sort(key=lambda o: (o[0], o[1]))
    return m, n, [(i, j, v) for j, i, v in obs]


@pytest.mark.parametrize("threads", ["1", "5"])
@pytest.mark.parametrize("header", [True, False])
def test_large_shuffled_file_matches_restatement(tmp_path, threads, header):
    """~2 MB of shuffled lines (several parser ranges), ragged whitespace, blank lines, CRLF."""
    os.environ["DFCG_IO_THREADS"] = threads
    try:
        rs = np.random.RandomState(5)
        m, n, N = 3000, 700, 90000
        cells = rs.choice(m * n, N, replace=False)
        vals = rs.standard_normal(N) * 10.0 ** rs.randint(-8, 8, N)
        seps = [" ", "\t", "  ", " \t "]
        lines = ["%% %d %d" % (m, n)] if header else []
        for c, v in zip(cells, vals):
            s = seps[c % 4]
            lines.append(("  " if c % 7 == 0 else "") + "%d%s%d%s%.17g" % (c % m, s, c // m, s, v) +
                         ("\r" if c % 5 == 0 else "") + (" " if c % 3 == 0 else ""))
            if c % 11 == 0:
                lines.append("")
        text = "\n".join(lines) + ("\n" if header else "")
        assert len(text) > (1 << 20)
        o = P.parse_triplets(text)
        rm, rn, rent = _ref_load(text.replace("\r", ""))
        assert (o.m, o.n) == (rm, rn)
        assert entries(o) == rent
        path = tmp_path / "big.txt"
        path.write_text(text)
        assert entries(P.load_triplets(path)) == rent
    finally:
        del os.environ["DFCG_IO_THREADS"]


def test_first_error_in_file_order_across_ranges():
    """Errors in two parser ranges: the earlier line wins, with its global line number."""
    os.environ["DFCG_IO_THREADS"] = "4"
    try:
        lines = ["% 100000 50"] + ["%d %d 1.0" % (i, i % 50) for i in range(100000)]
        lines[90001] = "7 7 7 extra"      # line 90002: trailing tokens
        lines[20000] = "200000 3 1.0"     # line 20001: outside the declared dims
        text = "\n".join(lines) + "\n"
        assert len(text) > (1 << 20)
        with pytest.raises(IndexError, match="line 20001: index outside declared 100000x50"):
            P.parse_triplets(text)
        lines[20000] = "5 x 1.0"
        with pytest.raises(P.ParseError) as e:
            P.parse_triplets("\n".join(lines) + "\n")
        assert e.value.line == 20001
        lines[20000] = "5 5 1.0"
        with pytest.raises(P.ParseError) as e:
            P.parse_triplets("\n".join(lines) + "\n")
        assert e.value.line == 90002 and "trailing tokens" in str(e.value)
    finally:
        del os.environ["DFCG_IO_THREADS"]


def test_load_feeds_the_d_step(tmp_path):
    """A generated instance saved and reloaded is the same ObservedMatrix (same D-step output)."""
    _, obs = P.gen_mc_instance(300, 200, 3, 12000, 0.1, 3)
    path = tmp_path / "inst.txt"
    P.save_triplets(path, obs)
    back = P.load_triplets(path)
    assert (back.m, back.n) == (obs.m, obs.n)
    assert np.array_equal(back.rows, obs.rows) and np.array_equal(back.cols, obs.cols)
    assert np.array_equal(back.vals, obs.vals)
    g = P.partition_columns(3, 0xDFC0000000000001, 200, 4)
    a, b = P.extract_columns(obs, g[1]), P.extract_columns(back, g[1])
    assert np.array_equal(a.vals, b.vals) and np.array_equal(a.rows, b.rows)


def test_missing_file():
    with pytest.raises(P.DfcError, match="cannot open"):
        P.load_triplets("/nonexistent/dir/x.txt")


# ---- fuzz: the parser against a character-level restatement of the istream extraction
import random  # noqa: E402
import re  # noqa: E402

def _istream_int(s, pos):
    # mimic istream >> long: skip ws, optional sign, digits
    n=len(s)
    while pos<n and s[pos] in ' \t\r\v\f\n': pos+=1
    q=pos
    if q<n and s[q] in '+-': q+=1
    d=q
    while q<n and s[q].isdigit(): q+=1
    if q==d: return None,pos
    return int(s[pos:q]), q
def _istream_dbl(s,pos):
    n=len(s)
    while pos<n and s[pos] in ' \t\r\v\f\n': pos+=1
    m=re.match(r'[+-]?(\d+\.?\d*|\.\d+)([eE][+-]?\d+)?', s[pos:])
    if not m: return None,pos
    # "1e" -> failure
    rest=s[pos+m.end():]
    if re.match(r'[eE]', rest): return None,pos
    v=float(m.group(0))
    if v in (float('inf'),float('-inf')): return None,pos
    return v,pos+m.end()
def _fuzz_ref(text, one_based):
    base=1 if one_based else 0
    m=n=-1; obs=[]; seen=False
    for ln,line in enumerate(text.split('\n'),1):
        toks=line.split()
        if not toks: continue
        if toks[0]=='%':
            if seen or m>=0: return ('parse',ln)
            p=line.index('%')+1
            a,p=_istream_int(line,p)
            if a is None: return ('parse',ln)
            b,p=_istream_int(line,p)
            if b is None or a<1 or b<1: return ('parse',ln)
            if line[p:].strip(): return ('parse',ln)
            m,n=a,b; continue
        i,p=_istream_int(line,0)
        if i is None: return ('parse',ln)
        j,p=_istream_int(line,p)
        if j is None: return ('parse',ln)
        v,p=_istream_dbl(line,p)
        if v is None: return ('parse',ln)
        if line[p:].strip(): return ('parse',ln)
        i-=base; j-=base
        if i<0 or j<0: return ('parse',ln)
        if m>=0 and (i>=m or j>=n): return ('range',ln)
        seen=True; obs.append((j,i,v))
    if m<0:
        if not obs: return ('inval',0)
        m=max(o[1] for o in obs)+1; n=max(o[0] for o in obs)+1
    obs.sort(key=lambda o:(o[0],o[1]))
    for a,b in zip(obs,obs[1:]):
        if a[0]==b[0] and a[1]==b[1]: return ('inval',0)
    return ('ok',(m,n,[(i,j,v) for j,i,v in obs]))


def _fuzz_ours(text, one_based):
    try:
        o = P.parse_triplets(text, one_based)
        return ('ok', (o.m, o.n, entries(o)))
    except P.ParseError as e:
        return ('parse', e.line)
    except IndexError as e:
        return ('range', int(re.match(r'line (\d+)', str(e)).group(1)))
    except ValueError:
        return ('inval', 0)


def test_fuzz_error_class_and_line_match_restatement():
    """Random small inputs built from valid and malformed fragments: the same outcome (matrix,
    or error class and line number) as load_triplets' istream logic (matrix_io.hpp:127-170)."""
    random.seed(1)
    frag = ['0', '1', '2', '3', '7', '-1', '+2', '1.5', '-.5', '2.', '1e2', '1e', 'x', '%', '% 4 4', '% 3', '  ',
            '\t', '9 9', 'inf', '0x1', '1e400', '3 3 3', '4 0 1 z', '']
    for _ in range(4000):
        lines = []
        for _ in range(random.randint(0, 6)):
            k = random.randint(0, 4)
            sep = random.choice([' ', '\t', '']) if random.random() < 0.5 else ' '
            lines.append(sep.join(random.choice(frag) for _ in range(k)))
        text = '\n'.join(lines) + random.choice(['', '\n'])
        ob = random.random() < 0.3
        assert _fuzz_ref(text, ob) == _fuzz_ours(text, ob), repr(text)
