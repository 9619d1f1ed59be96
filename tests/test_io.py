"""Reference-compatible I/O: the particle text format of
geometry.cpp:128-159 and the CostLedger JSON / CSV layout of ledger.cpp:56-86,
checked against the compiled reference (oracle/_ref)."""
import json
import os

import numpy as np
import pytest

from paper_2006_15367_b200 import io as hio


def _particles(n=257, seed=3):
    rng = np.random.default_rng(seed)
    pos = rng.standard_normal((n, 3)) * np.array([1e-3, 7.0, 1e5])
    q = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    pos[0] = [0.1, -0.0, 1e-300]  # awkward values survive the round trip
    q[0] = complex(1.0 / 3.0, -2.0 ** -1074)
    return pos, q


def test_particle_files_byte_identical_with_reference(tmp_path, refo):
    pos, q = _particles()
    ours, theirs = str(tmp_path / "ours.txt"), str(tmp_path / "ref.txt")
    hio.write_particles(ours, pos, q, "seeded test particles")
    refo.write_particles(theirs, pos, np.stack([q.real, q.imag], -1), "seeded test particles")
    assert open(ours).read() == open(theirs).read()
    # cross reads, bit-exact
    p2, q2 = refo.read_particles(ours)
    assert np.array_equal(p2, pos) and np.array_equal(q2[:, 0] + 1j * q2[:, 1], q)
    p3, q3 = hio.read_particles(theirs)
    assert np.array_equal(p3, pos) and np.array_equal(q3, q)


def test_particle_reader_comments_blank_lines_and_errors(tmp_path, refo):
    good = tmp_path / "good.txt"
    good.write_text("# header\n\n1 2 3 4 5\n# mid\n6 7 8 9 10 extra\n")
    p, q = hio.read_particles(str(good))
    rp, rq = refo.read_particles(str(good))
    assert np.array_equal(p, rp) and np.array_equal(q, rq[:, 0] + 1j * rq[:, 1])
    bad = tmp_path / "bad.txt"
    bad.write_text("1 2 3 4 5\n1 2 3 x 5\n")
    with pytest.raises(RuntimeError) as ours:
        hio.read_particles(str(bad))
    with pytest.raises(Exception) as theirs:
        refo.read_particles(str(bad))
    assert str(ours.value) == f"{bad}:2: expected 'x y z re im'"
    assert str(ours.value) in str(theirs.value)
    with pytest.raises(RuntimeError, match="cannot open particle file"):
        hio.read_particles(str(tmp_path / "missing.txt"))


def test_ledger_layout():
    ph = {"Tbuild": 1.5, "C2M": 1.25, "M2M": 7.0, "M2L": 12.0, "L2L": 8.0, "L2T": 1.5, "Near": 0.75, "total": 30.0}
    ranks = hio.ledger_ranks([ph, ph], flops={"m2l": 3 * 10 ** 11}, messages=[{"m2l": 0}, {"m2l": 4}],
                             bytes_=[{"m2l": 0}, {"m2l": 4096}], mem_peak={"temporaries": 123})
    j = json.loads(hio.ledger_json(ranks))
    assert j["time_basis"] == "wall" and len(j["ranks"]) == 2
    for e in j["ranks"]:
        assert sorted(e["phases"]) == sorted(hio.PHASES)
        assert sorted(e["mem_peak"]) == sorted(hio.MEM_CLASSES)
        for c in e["phases"].values():
            assert sorted(c) == ["bytes", "flops", "messages", "seconds"]
    assert j["ranks"][0]["phases"]["m2l"]["seconds"] == pytest.approx(0.012)
    assert j["ranks"][1]["phases"]["m2l"]["bytes"] == 4096
    csv = hio.ledger_csv(ranks).splitlines()
    assert csv[0] == "rank,phase,flops,messages,bytes,seconds"
    assert len(csv) == 1 + 2 * len(hio.PHASES)
    assert csv[1 + hio.PHASES.index("m2l")] == "0,m2l,300000000000,0,0,0.012"
