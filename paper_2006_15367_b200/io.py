"""Reference-compatible I/O and cost reporting.

* read_particles / write_particles: the reference's particle text format
  (proj/src/geometry.cpp:128-159): '#' comment lines, one particle per line
  as 'x y z re im', written with 17 significant digits.  Same error text.
* ledger_json / ledger_csv: the reference's CostLedger layout
  (proj/src/ledger.cpp:56-86): per rank, per phase {flops, messages, bytes,
  seconds} and per memory class peak bytes, so studies that read the
  reference's ledgers read ours.  Seconds are the engine's device times;
  flops follow paper_2006_15367_b200.accounting.
"""
from __future__ import annotations

import json

import numpy as np

# hfmm::Phase order and names (proj/include/hfmm/ledger.hpp:12, ledger.cpp:9-20)
PHASES = ("setup", "c2m", "m2m", "m2l", "l2l", "l2o", "near")
# hfmm::MemClass (ledger.hpp:17, ledger.cpp:22-30)
MEM_CLASSES = ("tree_storage", "translation_operators", "comm_buffers", "temporaries")
# engine timing slots (hfmm_gpu_timing.ms) -> ledger phases
_FROM_ENGINE = {"Tbuild": "setup", "C2M": "c2m", "M2M": "m2m", "M2L": "m2l", "L2L": "l2l", "L2T": "l2o",
                "Near": "near"}


def read_particles(path: str):
    """hfmm::read_particles: -> (positions (n, 3) float64, intensities (n,) complex128)."""
    xyz, q = [], []
    try:
        fh = open(path)
    except OSError:
        raise RuntimeError(f"cannot open particle file: {path}") from None
    with fh:
        for lineno, line in enumerate(fh, 1):
            line = line.rstrip("\n")
            if not line or line[0] == "#":
                continue
            parts = line.split()
            try:
                vals = [float(v) for v in parts[:5]]
                if len(vals) < 5:
                    raise ValueError
            except ValueError:
                raise RuntimeError(f"{path}:{lineno}: expected 'x y z re im'") from None
            xyz.append(vals[:3])
            q.append(complex(vals[3], vals[4]))
    return np.asarray(xyz, dtype=np.float64).reshape(-1, 3), np.asarray(q, dtype=np.complex128)


def write_particles(path: str, positions, intensities, header_comment: str = "") -> None:
    """hfmm::write_particles: 17 significant digits (std::ostream precision 17)."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    q = np.asarray(intensities, dtype=np.complex128).reshape(-1)
    if pos.shape[0] != q.shape[0]:
        raise ValueError("write_particles: positions and intensities differ in length")
    try:
        fh = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot open particle file for write: {path}") from None
    with fh:
        if header_comment:
            fh.write(f"# {header_comment}\n")
        for (x, y, z), c in zip(pos, q):
            fh.write(f"{x:.17g} {y:.17g} {z:.17g} {c.real:.17g} {c.imag:.17g}\n")


def ledger_ranks(phase_ms_per_rank, flops=None, messages=None, bytes_=None, mem_peak=None):
    """Ledger entries from per-rank engine timings (dicts like RankEngine.last_timing()[0]).

    flops / messages / bytes_: optional dicts ledger-phase -> value (same for every
    rank unless given as a list of dicts); mem_peak: dict class -> bytes (or list).
    """
    def pick(v, r):
        return v[r] if isinstance(v, (list, tuple)) else v

    ranks = []
    for r, ph in enumerate(phase_ms_per_rank):
        e = {"phases": {}, "mem_peak": {}}
        for p in PHASES:
            e["phases"][p] = {"flops": 0, "messages": 0, "bytes": 0, "seconds": 0.0}
        for k, v in ph.items():
            if k in _FROM_ENGINE:
                e["phases"][_FROM_ENGINE[k]]["seconds"] = float(v) / 1e3
        for key, src in (("flops", flops), ("messages", messages), ("bytes", bytes_)):
            d = pick(src, r) if src is not None else None
            for p, v in (d or {}).items():
                e["phases"][p][key] = int(v)
        mp = pick(mem_peak, r) if mem_peak is not None else {}
        for c in MEM_CLASSES:
            e["mem_peak"][c] = int((mp or {}).get(c, 0))
        ranks.append(e)
    return ranks


def ledger_json(ranks, time_basis: str = "wall") -> str:
    """CostLedger::to_json layout (ledger.cpp:56-74), 2-space indent."""
    return json.dumps({"ranks": ranks, "time_basis": time_basis}, indent=2)


def ledger_csv(ranks) -> str:
    """CostLedger::to_csv layout (ledger.cpp:76-86)."""
    out = ["rank,phase,flops,messages,bytes,seconds"]
    for r, e in enumerate(ranks):
        for p in PHASES:
            c = e["phases"][p]
            out.append(f"{r},{p},{c['flops']},{c['messages']},{c['bytes']},{c['seconds']:g}")
    return "\n".join(out) + "\n"


def evaluation_ledger(setup, phase_ms, exchange=None) -> list:
    """Ledger of one single-rank evaluation: device seconds per phase and the
    algorithmic flops of paper_2006_15367_b200.accounting."""
    from .accounting import phase_accounting
    acc, _ = phase_accounting(setup)
    names = {"C2M": "c2m", "M2M": "m2m", "M2L": "m2l", "L2L": "l2l", "L2T": "l2o", "Near": "near"}
    flops = {names[k]: v[0] for k, v in acc.items() if k in names}
    return ledger_ranks([phase_ms], flops=flops, messages=(exchange or {}).get("messages"),
                        bytes_=(exchange or {}).get("bytes"))
