"""Host ingestion (csrc/ingest.cpp) vs the reference's fixtures and unit tests:
the 5 hand-tallied PTX fixtures of acceptance criterion 7
(acceptance_main.cpp:330-351, copied as data into tests/golden/ptx/) and the cases
of test_ptx_features.cpp / test_telemetry.cpp.  Host code: runs on CPU."""

import json
import os

import numpy as np
import pytest

from paper_2407_13096_b200 import DsoError, ErrorKind
from paper_2407_13096_b200.ingest import ingest_corpus, load_dcgm_samples, parse_ptx, ptx_csr

HERE = os.path.join(os.path.dirname(__file__), "golden", "ptx")
CATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "categories.json")))


def names_of():
    c = CATS
    return list(c["instr"]), list(c["dtype"]), list(c["memspace"])


def tally(counts):
    ins, dt, ms = names_of()
    out = ({}, {}, {})
    for r, v in enumerate(counts):
        if v:
            if r < 101:
                out[0][ins[r]] = int(v)
            elif r < 118:
                out[1][dt[r - 101]] = int(v)
            else:
                out[2][ms[r - 118]] = int(v)
    return out


def wrap(body):
    return ".version 7.0\n.target sm_70\n.visible .entry k()\n{\n" + body + "\n}\n"


def test_categories_shape():
    ins, dt, ms = names_of()
    assert len(ins) == 101 and len(dt) == 17 and len(ms) == 8
    assert ins[-1] == dt[-1] == ms[-1] == "other"


@pytest.mark.parametrize("name", ["saxpy_basic.ptx", "predicated.ptx", "vector_memory.ptx",
                                  "multi_kernel.ptx", "exotic_ops.ptx"])
def test_fixture_tallies(name):
    g = json.load(open(os.path.join(HERE, "golden_tallies.json")))["fixtures"][name]
    ks = parse_ptx(open(os.path.join(HERE, name)).read())
    assert len(ks) == g["kernels"]
    ins, dt, ms = tally(ks[g["index"]][1])
    assert ins == g["instr"] and dt == g["dtype"] and ms == g["memspace"]


def test_multi_kernel_order_and_decl():
    ks = parse_ptx(open(os.path.join(HERE, "multi_kernel.ptx")).read())
    assert [k[0] for k in ks] == ["alpha", "beta", "gamma_decl"]
    assert ks[1][2] == 0 and ks[2][2] == 0  # empty body, declaration


def test_hand_counts():
    k = parse_ptx(wrap("add.s32 %r1,%r2,%r3; bra L1;"))[0]
    ins, dt, ms = tally(k[1])
    assert ins == {"add": 1, "bra": 1} and dt == {".s32": 1} and ms == {} and k[2] == 2
    k = parse_ptx(wrap(""))[0]
    assert k[2] == 0 and not k[1].any()
    k = parse_ptx(wrap("ld.shared.f64 %fd1, [a];\nld.shared.f64 %fd2, [b];\n"
                       "st.global.f64 [c], %fd1;\nld.tex.u32 %r1, [t];"))[0]
    ins, dt, ms = tally(k[1])
    assert ms == {".shared": 2, ".global": 1, "other": 1} and dt[".f64"] == 3


def test_guards_labels_directives():
    k = parse_ptx(wrap(".reg .b32 %r<4>;\nL0:\n@%p1 bra L0;\n@!%p2 add.u32 %r1,%r2,%r3;\n"
                       "{ mov.u32 %r1, %r2; }\n$L__x: sub.s64 %rd1, %rd2, %rd3;"))[0]
    ins, dt, _ = tally(k[1])
    assert ins == {"bra": 1, "add": 1, "mov": 1, "sub": 1}
    assert dt == {".u32": 2, ".s64": 1}


def test_malformed():
    with pytest.raises(DsoError) as e:
        parse_ptx(".entry broken\n{\n  add.s32 %r1,%r2,%r3;\n")
    assert e.value.kind == ErrorKind.MalformedPtx and "line 2" in str(e.value)
    with pytest.raises(DsoError) as e:
        parse_ptx("/* never closed")
    assert e.value.kind == ErrorKind.MalformedPtx


def test_entry_count_and_roundtrip():
    rng = np.random.default_rng(13)
    pool = ["add.s32 %r1,%r2,%r3;", "ld.global.f32 %f1,[%rd1];", "st.shared.f64 [%rd1],%fd1;",
            "fma.rn.f32 %f1,%f2,%f3,%f4;", "bogusop.u16 %r1;", "bra L0;"]
    for _ in range(20):
        n = int(rng.integers(0, 6))
        src = ".version 7.0\n" + "".join(
            f".visible .entry k{i}()\n{{\n" + "".join(pool[int(j)] + "\n" for j in
                                                     rng.integers(0, 6, int(rng.integers(0, 30))))
            + "}\n" for i in range(n))
        ks = parse_ptx(src)
        assert len(ks) == n
        names, rp, ent = ptx_csr(src)
        assert len(names) == n and int(rp[-1]) == len(ent)
        for k, (_, c, _) in enumerate(ks):
            dense = np.zeros(126, np.uint64)
            for e in ent[int(rp[k]):int(rp[k + 1])]:
                dense[int(e) & 127] += int(e) >> 7
            np.testing.assert_array_equal(dense, c)


def test_dcgm():
    H = "timestamp,SMACT,SMOCC,TENSO,DRAMA,FP64A,FP32A,FP16A,INTAC\n"
    v = load_dcgm_samples(H + "0,0.8,0,0,0,0,0,0,0\n")
    assert v[0] == pytest.approx(0.8) and v[1] == 0.0
    v = load_dcgm_samples(H + "0,0.6,0.1,0,0.2,0,0.5,0,0.3\n1,0.8,0.3,0,0.4,0,0.7,0,0.1\n")
    np.testing.assert_allclose(v[[0, 1, 3, 5, 7]], [0.7, 0.2, 0.3, 0.6, 0.2])
    v = load_dcgm_samples(H.replace("\n", "\r\n") + "0,0.4,0,0,0,0,0,0,0\r\n")
    assert v[0] == pytest.approx(0.4)
    for bad, kind in ((H + "0,0.5,0,0,1.3,0,0,0,0\n", ErrorKind.OutOfRange),
                      (H, ErrorKind.EmptyTrace), ("timestamp,SMACT\n0,0.5\n", ErrorKind.SchemaMismatch),
                      (H + "0,0.5,0,0\n", ErrorKind.SchemaMismatch),
                      (H + "0,x,0,0,0,0,0,0,0\n", ErrorKind.SchemaMismatch)):
        with pytest.raises(DsoError) as e:
            load_dcgm_samples(bad)
        assert e.value.kind == kind
    with pytest.raises(DsoError) as e:
        load_dcgm_samples(H + "0,0.5,0,0,1.3,0,0,0,0\n")
    assert "row 1" in str(e.value)


def test_ingest_corpus():
    texts = [open(os.path.join(HERE, f)).read() for f in sorted(os.listdir(HERE)) if f.endswith(".ptx")]
    H = "timestamp,SMACT,SMOCC,TENSO,DRAMA,FP64A,FP32A,FP16A,INTAC\n"
    dc = [H + f"0,0.{i + 1},0.2,0,0.3,0,0.4,0,0.5\n" for i in range(len(texts))]
    names, rp, ent, dcgm = ingest_corpus(texts, dc, threads=4)
    assert len(names) == len(texts) and dcgm.shape == (8, len(texts)) and rp[-1] == len(ent)
