"""Trace ingestion (TraceStream / TraceSchema / load_schema, workload.hpp:137-300)
on the host: the reference's own trace tests (tests/test_workload.cpp:179-281)
restated, a ZipfStream round trip, and randomized traces -- malformed tokens,
signs, overflow, blank lines, duplicates, schemas, oversized samples, files
large enough for the parallel parser -- checked byte for byte (batches, counts,
warning text, error message) against the compiled reference (oracle/_ref)."""
import io
import os

import numpy as np
import pytest

from helpers import canon_equal


def cfg_of(edx, n, m, cap=None):
    return edx.ClusterConfig(n=n, m=m, bandwidths_bps=[5e9] * n, d_tran_bytes=2048,
                             cache_capacity=cap if cap is not None else 64, alpha=0.0)


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode("latin-1") if isinstance(text, str) else text)
    return str(p)


def batches(ts):
    out = []
    for ids, offs in ts:
        out.append([ids[offs[i]:offs[i + 1]].tolist() for i in range(len(offs) - 1)])
    return out


# ---- tests/test_workload.cpp:179-259, restated
def test_two_lines_two_workers_one_iteration(edx, tmp_path):
    ts = edx.TraceStream(write(tmp_path, "a.txt", "1 2 3\n4 5 6\n"), cfg_of(edx, 2, 1))
    assert batches(ts) == [[[1, 2, 3], [4, 5, 6]]]
    assert ts.dropped_samples() == 0 and ts.iterations() == 1 and ts.max_sample_len() == 3


def test_duplicates_collapse(edx, tmp_path):
    ts = edx.TraceStream(write(tmp_path, "b.txt", "3 3 7\n8 9 10\n"), cfg_of(edx, 2, 1))
    assert batches(ts)[0][0] == [3, 7]


def test_trailing_partial_iteration_dropped_with_warning(edx, tmp_path):
    w = io.StringIO()
    p = write(tmp_path, "c.txt", "1\n2\n3\n")
    ts = edx.TraceStream(p, cfg_of(edx, 2, 1), warnings=w)
    assert len(batches(ts)) == 1 and ts.dropped_samples() == 1
    assert w.getvalue() == f"warning: {p}: dropping 1 trailing sample(s) of a partial iteration\n"


def test_malformed_line_named(edx, tmp_path):
    p = write(tmp_path, "d.txt", "1 2\nx 4\n")
    with pytest.raises(edx.EdxRuntimeError, match=f"^{p}:2: malformed id 'x'$"):
        edx.TraceStream(p, cfg_of(edx, 2, 1))


def test_empty_trace_rejected(edx, tmp_path):
    p = write(tmp_path, "e.txt", "")
    with pytest.raises(edx.EdxRuntimeError, match="trace file holds no samples"):
        edx.TraceStream(p, cfg_of(edx, 2, 1))
    with pytest.raises(edx.EdxRuntimeError, match="cannot open trace file"):
        edx.TraceStream(str(tmp_path / "missing.txt"), cfg_of(edx, 2, 1))


def test_schema_offsets_flatten(edx, tmp_path):
    schema = edx.load_schema(write(tmp_path, "s.txt", "users 10\nitems 20\nads 5\n"))
    assert schema.total_embeddings() == 35
    ts = edx.TraceStream(write(tmp_path, "f.txt", "1 2 3\n9 19 4\n"), cfg_of(edx, 2, 1), schema)
    assert batches(ts) == [[[1, 12, 33], [9, 29, 34]]]
    bad = write(tmp_path, "g.txt", "10 0 0\n0 0 0\n")
    with pytest.raises(edx.EdxRuntimeError, match=":1: row id 10 exceeds table 'users'"):
        edx.TraceStream(bad, cfg_of(edx, 2, 1), schema)
    bad = write(tmp_path, "h.txt", "1 2\n3 4\n")
    with pytest.raises(edx.EdxRuntimeError, match=":1: expected 3 fields per schema, got 2"):
        edx.TraceStream(bad, cfg_of(edx, 2, 1), schema)


def test_schema_without_tables(edx, tmp_path):
    """A TraceSchema with no tables is still a schema: every id line has too
    many fields (workload.hpp:227-232 with an empty offset list)."""
    p = write(tmp_path, "z.txt", "\n1 2 3\n")
    with pytest.raises(edx.EdxRuntimeError, match=":2: expected 0 fields per schema, got 3"):
        edx.TraceStream(p, cfg_of(edx, 2, 1), edx.TraceSchema())


def test_oversized_sample_rejected(edx, tmp_path):
    p = write(tmp_path, "i.txt", "1 2 3\n4 5 6\n7 8 9\n10 11 12\n")
    with pytest.raises(edx.EdxRuntimeError,
                       match=r":1: sample of 3 ids cannot fit the per-worker cache \(capacity 4, m 2\)"):
        edx.TraceStream(p, cfg_of(edx, 2, 2, cap=4))


def test_zipf_round_trip(edx, tmp_path):
    """test_workload.cpp:261-281: a generated stream written as a trace reads back."""
    cfg = cfg_of(edx, 2, 2)
    z = edx.ZipfStream(300, 4, 1.05, 3, 17, cfg.samples_per_iteration())
    want = [ids.reshape(-1, 4).tolist() for ids in z]
    text = "".join(" ".join(map(str, s)) + "\n" for b in want for s in b)
    assert text.count("\n") == 12
    ts = edx.TraceStream(write(tmp_path, "rt.txt", text), cfg)
    assert batches(ts) == want
    ts.reset()
    assert batches(ts) == want


# ---- randomized parity against the compiled reference
def py_dump(edx, path, schema_path, n, m, cap):
    try:
        schema = edx.load_schema(schema_path) if schema_path else None
        w = io.StringIO()
        ts = edx.TraceStream(path, cfg_of(edx, n, m, cap), schema, warnings=w)
    except edx.EdxRuntimeError as e:
        return False, str(e)
    lines = [f"iterations {ts.iterations()} dropped {ts.dropped_samples()} "
             f"max {ts.max_sample_len()}\n"]
    for b in batches(ts):
        lines += [" ".join(map(str, s)) + "\n" for s in b]
    return True, "".join(lines) + w.getvalue()


TOKENS_GOOD = ["0", "1", "7", "+5", "007", "-1", "-4294967297", "4294967296", "4294967301",
               "18446744073709551615", "99"]
TOKENS_BAD = ["x", "1x", "0x1f", "-", "+", "+-1", "18446744073709551616", "1.5", "1e3"]
SEPS = [" ", "  ", "\t", " \r", "\v", "\f"]


def random_trace(rng, lines, width, bad_rate, id_hi):
    out = []
    for _ in range(lines):
        if rng.random() < 0.05:
            out.append(rng.choice(["", "   ", "\t\r"]))
            continue
        toks = []
        for _ in range(int(rng.integers(1, width + 1))):
            r = rng.random()
            if r < bad_rate:
                toks.append(str(rng.choice(TOKENS_BAD)))
            elif r < 0.1:
                toks.append(str(rng.choice(TOKENS_GOOD)))
            else:
                toks.append(str(int(rng.integers(0, id_hi))))
        lead = rng.choice(["", " ", "\t"])
        out.append(lead + "".join(t + str(rng.choice(SEPS)) for t in toks[:-1]) + toks[-1])
    text = "\n".join(out)
    if rng.random() < 0.7:
        text += "\n"
    return text


@pytest.mark.parametrize("seed", range(40))
def test_random_traces_match_reference(edx, ref, tmp_path, seed):
    rng = np.random.default_rng(seed)
    n, m = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    lines = int(rng.integers(0, 40))
    bad = [0.0, 0.0, 0.002, 0.02][seed % 4]
    width = int(rng.integers(1, 8)) if seed % 5 else 90  # > 64: hash-set dedup path
    cap = int(rng.choice([0, 6, 64, 10_000]))
    text = random_trace(rng, lines, width, bad, 40 if seed % 3 else 5)
    path = write(tmp_path, "t.txt", text)
    got = py_dump(edx, path, None, n, m, cap)
    assert got == ref.trace_dump(path, None, n, m, cap)


@pytest.mark.parametrize("seed", range(20))
def test_random_schema_traces_match_reference(edx, ref, tmp_path, seed):
    rng = np.random.default_rng(1000 + seed)
    k = int(rng.integers(1, 5))
    sizes = [int(rng.integers(1, 30)) for _ in range(k)]
    sch = "".join(f"t{i} {s}\n" for i, s in enumerate(sizes))
    if seed % 7 == 3:
        sch += "\n  \n"
    spath = write(tmp_path, "s.txt", sch)
    rows = []
    for _ in range(int(rng.integers(1, 20))):
        kk = k if rng.random() > 0.03 else k + 1
        rows.append(" ".join(str(int(rng.integers(0, (sizes[i % k] + (1 if rng.random() < 0.01
                                                                       else 0)))))
                             for i in range(kk)))
    path = write(tmp_path, "t.txt", "\n".join(rows) + "\n")
    n, m = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    assert py_dump(edx, path, spath, n, m, 0) == ref.trace_dump(path, spath, n, m, 0)


@pytest.mark.parametrize("text", ["a 5\n", "a 0\n", "a\n", "a x\n", "a +3\n", "a -1\n",
                                  "a 18446744073709551616\n", "a 7junk\n", "\n\n", "",
                                  "a 3\nb\n", "  a\t4 extra\n"])
def test_schema_parsing_matches_reference(edx, ref, tmp_path, text):
    spath = write(tmp_path, "s.txt", text)
    path = write(tmp_path, "t.txt", "0\n")
    assert py_dump(edx, path, spath, 1, 1, 0) == ref.trace_dump(path, spath, 1, 1, 0)


def test_large_trace_parallel_parser_matches_reference(edx, ref, tmp_path):
    """A multi-MiB trace (parsed in newline-aligned chunks on every host
    thread): batches, then the first error in file order when late lines
    fail in several chunks."""
    rng = np.random.default_rng(7)
    R, L = 400_000, 12
    ids = rng.integers(0, 50_000, size=(R, L))
    text = "\n".join(" ".join(map(str, r)) for r in ids.tolist()) + "\n"
    path = write(tmp_path, "big.txt", text)
    got = py_dump(edx, path, None, 7, 9, 0)
    assert got[0] and got == ref.trace_dump(path, None, 7, 9, 0)
    lines = text.split("\n")
    for at in (R - 5, R // 2 + 3, R // 3):
        lines[at] = lines[at] + " bad" + str(at)
    path = write(tmp_path, "big_bad.txt", "\n".join(lines))
    got = py_dump(edx, path, None, 7, 9, 0)
    assert not got[0] and f":{R // 3 + 1}: malformed id 'bad{R // 3}'" in got[1]
    assert got == ref.trace_dump(path, None, 7, 9, 0)


# ---- a trace driving the device engine: ragged samples, bit-exact vs the oracle
@pytest.mark.gpu
@pytest.mark.parametrize("n,m,alpha,maxlen,V,schema", [(8, 16, 0.5, 40, 3000, False),
                                                       (4, 32, 0.0, 26, 2000, True),
                                                       (16, 8, 1.0, 70, 5000, False)])
def test_trace_drives_engine(gpu, oracle, pyoracle, tmp_path, n, m, alpha, maxlen, V, schema):
    """Ragged trace samples (1..maxlen ids with duplicates, blank lines, a
    dropped partial iteration) parsed by TraceStream and run through
    SimState.iterate: decisions, reports, expected costs and the final state
    equal the reference iteration on the same batches."""
    edx = gpu
    rng = np.random.default_rng(n * 1000 + m)
    R = n * m
    iters = 6
    sch = None
    if schema:  # 26 tables, one field each: fixed-width lines flattened by the schema
        sizes = [int(s) for s in rng.integers(20, 150, size=26)]
        spath = write(tmp_path, "s.txt", "".join(f"f{i} {s}\n" for i, s in enumerate(sizes)))
        sch = edx.load_schema(spath)
        V = sch.total_embeddings()
        rows = [" ".join(str(int(min(rng.zipf(1.3), s) - 1)) for s in sizes)
                for _ in range(R * iters + 3)]
    else:
        rows = []
        for _ in range(R * iters + 5):
            k = int(rng.integers(1, maxlen + 1))
            rows.append(" ".join(str(int(x) % V) for x in rng.zipf(1.2, size=k)))
    rows.insert(7, "   ")
    path = write(tmp_path, "t.txt", "\n".join(rows) + "\n")
    bw = [5e9] * (n // 2) + [5e8] * (n - n // 2)
    cap = m * maxlen + 50
    c = edx.ClusterConfig(n=n, m=m, bandwidths_bps=bw, d_tran_bytes=2048, cache_capacity=cap,
                          alpha=alpha)
    ts = edx.TraceStream(path, c, sch, warnings=io.StringIO())
    assert ts.iterations() == iters and ts.dropped_samples() in (3, 5)
    eng = edx.SimState(c, id_space=V, max_batch_ids=R * max(maxlen, 26))
    sim = oracle.sim(pyoracle.Cfg(n, m, bw, cap=cap, alpha=alpha))
    for it, (ids, offs) in enumerate(ts):
        dec, rep = eng.iterate(ids, offs)
        wdec, wexp, wrep, _ = sim.iteration(ids, offs)
        assert (dec == wdec).all(), f"iter {it}: decision"
        assert rep.as_dict() == wrep, f"iter {it}: report"
        assert rep.expected_cost_s == wexp, f"iter {it}: expected cost"
    msg = canon_equal(eng.canonical_state(), sim.canonical_state())
    assert not msg, msg
    eng.validate_consistency()
