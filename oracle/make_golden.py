"""Generate tests/golden/*.npz by running the REFERENCE implementation (hexmc) in this container.

Usage (in the build container, where /root/reference exists; never on the GPU box):
    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

The reference is imported from /root/reference/pkg/src (read-only; numba cache redirected).
Fixtures are small: masks, selected H/S matrices, eigenvalues, per-sample curves, level moments,
plus the reference's own end-to-end artifacts (pkg/frontend/fixtures/{rates,bilevel}) parsed into
arrays.  Test infrastructure only.
"""

from __future__ import annotations

import csv
import json
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

import hexmc  # noqa: E402
from hexmc import (  # noqa: E402
    EnergyGrid,
    GrapheneNNModel,
    SmoothingSpec,
    assemble_bloch,
    build_supercell,
    idos,
    idos_sharp,
    load_coupling_table,
    make_bz_grid,
    partition_quarters,
    solve_bands,
)
from hexmc.disorder import DefectConfiguration, SeedSpec, restrict, sample_defects  # noqa: E402
from hexmc.runner import Engine  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
TABLE = OUT / "synthetic_11band.tbc"


def key_words(key: int, nunits: int) -> np.ndarray:
    nw = (nunits + 63) // 64
    return np.array([(key >> (64 * i)) & ((1 << 64) - 1) for i in range(nw)], dtype=np.uint64)


def gen_rng():
    seeds = [2026, 2024, 123, 7, 0, 2**40 + 5]
    levels = [0, 1, 2, 3, 4, 10_004]
    reps = list(range(0, 40)) + [1000, 65535, 2**32 + 3]
    rows = []
    draws = []
    for s in seeds:
        for lv in levels:
            for r in reps:
                rows.append((s, lv, r))
                g = SeedSpec(s, lv, r).generator()
                draws.append(g.random(16))
    masks = {}
    g = GrapheneNNModel()
    for nu in (1, 2, 4, 8, 16, 32):
        sc = build_supercell(g.lattice_spec(), nu)
        ks = [sample_defects(sc, 0.05, SeedSpec(2026, 1 + (nu % 5), m)).key for m in range(24)]
        masks[f"graphene_nu{nu}"] = np.stack([key_words(k, sc.nunits) for k in ks])
    np.savez_compressed(
        OUT / "rng.npz",
        streams=np.array(rows, dtype=np.uint64),
        draws=np.array(draws),
        **masks,
    )


def gen_assembly():
    g = GrapheneNNModel()
    tab = load_coupling_table(TABLE)
    out = {}
    cases = [
        ("g2_v3", g, 2, frozenset({3}), (0.1, -0.2)),
        ("g1_gamma", g, 1, frozenset(), (0.0, 0.0)),
        ("g4_rand", g, 4, None, (0.31, 0.77)),
        ("g3_none", g, 3, frozenset(), (1.1, -0.4)),
        ("t2_v1", tab, 2, frozenset({1}), (0.2, 0.5)),
        ("t1_none", tab, 1, frozenset(), (0.4, -0.3)),
    ]
    for name, model, nu, vac, k in cases:
        sc = build_supercell(model.lattice_spec(), nu)
        if vac is None:
            cfg = sample_defects(sc, 0.2, SeedSpec(99, 1, 3))
        else:
            cfg = DefectConfiguration(sc, vac)
        pair = assemble_bloch(model, sc, cfg, k)
        out[f"{name}_H"] = pair.H
        out[f"{name}_S"] = pair.S
        out[f"{name}_k"] = np.array(k)
        out[f"{name}_mask"] = key_words(cfg.key, sc.nunits)
    np.savez_compressed(OUT / "assembly.npz", **out)


def gen_eigs_and_curves():
    g = GrapheneNNModel()
    tab = load_coupling_table(TABLE)
    out = {}
    # graphene nu=4 q=6 (config 1 shape), nu=8 q=4, nu=16 q=1 ; table nu=2 q=4, nu=4 q=2
    cases = [
        ("g4q6", g, 4, 6, 0.05, 10),
        ("g8q4", g, 8, 4, 0.05, 3),
        ("g16q1", g, 16, 1, 0.05, 2),
        ("t2q4", tab, 2, 4, 0.05, 4),
        ("t4q2", tab, 4, 2, 0.2, 2),
    ]
    lo_g, hi_g = -6.580201874549387, 14.863393148450246
    for name, model, nu, q, p, nsamp in cases:
        sc = build_supercell(model.lattice_spec(), nu)
        cell = hexmc.tbmodel.compile_cell(model, sc)
        bzr = make_bz_grid(model.lattice_spec(), nu, q, "reduced")
        bzf = make_bz_grid(model.lattice_spec(), nu, q, "full")
        if model is g:
            grid = EnergyGrid(lo_g, hi_g, 201)
        else:
            grid = EnergyGrid(-2.932 - 0.02, 4.740 + 0.02, 201)
        masks, eigs, curves, curves_full, sharp = [], [], [], [], []
        for m in range(nsamp):
            cfg = sample_defects(sc, p, SeedSpec(2026, 7, m))
            bands = solve_bands(model, sc, cfg, bzr, cell=cell)
            bands_f = solve_bands(model, sc, cfg, bzf, cell=cell)
            e = np.full((bzr.nk, cell.dim), np.nan)
            e[:, : bands.nbands] = bands.energies
            masks.append(key_words(cfg.key, sc.nunits))
            eigs.append(e)
            curves.append(idos(bands, grid, SmoothingSpec(0.01), sc.area).values)
            curves_full.append(idos(bands_f, grid, SmoothingSpec(0.01), sc.area).values)
            sharp.append(idos_sharp(bands, grid, sc.area).values)
        out[f"{name}_masks"] = np.stack(masks)
        out[f"{name}_eigs"] = np.stack(eigs)
        out[f"{name}_kpoints"] = bzr.kpoints
        out[f"{name}_curves"] = np.stack(curves)
        out[f"{name}_curves_full"] = np.stack(curves_full)
        out[f"{name}_sharp"] = np.stack(sharp)
        out[f"{name}_grid"] = np.array([grid.lo, grid.hi, grid.npoints])
        out[f"{name}_meta"] = np.array([nu, q])
    np.savez_compressed(OUT / "eigs_curves.npz", **out)


def gen_levels():
    g = GrapheneNNModel()
    eng = Engine(g, nq=16, delta=0.01, master_seed=2026, workers=1, bz_mode="reduced", energy_points=201)
    out = {"grid": np.array([eng.grid.lo, eng.grid.hi, eng.grid.npoints])}
    recs = []
    for level, (n, M) in enumerate(((4, 24), (8, 8)), start=1):
        s = eng.sample_level(level, n, M, 0.05, with_cv=level > 1)
        out[f"L{level}_mean"] = s.stats.mean
        out[f"L{level}_var"] = s.stats.sample_variance
        out[f"L{level}_full"] = s.full
        if s.cv is not None:
            out[f"L{level}_cv"] = s.cv
        recs.append([level, n, s.stats.q, M, s.stats.cache_hits])
    out["records"] = np.array(recs)
    tab = load_coupling_table(TABLE)
    et = Engine(tab, nq=4, delta=0.01, master_seed=2026, workers=1, bz_mode="reduced", energy_points=201,
                energy_range=(-2.932, 4.740))
    s = et.sample_level(1, 2, 6, 0.05, with_cv=False)
    out["table_L1_mean"] = s.stats.mean
    out["table_L1_full"] = s.full
    out["table_grid"] = np.array([et.grid.lo, et.grid.hi, et.grid.npoints])
    np.savez_compressed(OUT / "levels.npz", **out)


def read_csv_cols(path):
    with open(path) as fh:
        r = csv.reader(fh)
        header = next(r)
        rows = [[float(x) for x in row] for row in r]
    return header, np.array(rows)


def gen_fx():
    fx = REF / "frontend" / "fixtures"
    out = {}
    for run in ("rates", "bilevel"):
        for name in ("idos", "unperturbed", "slmc"):
            p = fx / run / f"{name}.csv"
            if p.exists():
                _, arr = read_csv_cols(p)
                out[f"{run}_{name}"] = arr
        levels = [json.loads(line) for line in open(fx / run / "levels.jsonl")]
        out[f"{run}_levels_json"] = np.array(json.dumps(levels))
        out[f"{run}_summary_json"] = np.array((fx / run / "summary.json").read_text())
    np.savez_compressed(OUT / "fx_reference_artifacts.npz", **out)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    if not TABLE.exists():
        TABLE.write_text((REF / "data" / "synthetic_11band.tbc").read_text())
    gen_rng()
    gen_assembly()
    gen_eigs_and_curves()
    gen_levels()
    gen_fx()
    print("golden fixtures written to", OUT)
