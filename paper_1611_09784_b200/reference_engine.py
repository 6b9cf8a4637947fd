"""The maintainer's drop-in for the reference package: its own Engine with only the batch seam replaced.

`cuda_engine_class(hexmc.runner.Engine)` returns a subclass of the REFERENCE Engine whose
`evaluate_masks` (runner.py:206-244) keeps the reference's dedup / placement loop verbatim but sends the
new jobs of each (n, q) group to one `hx_eval_idos_batch` call (libhx, sm_100a) instead of
`parallel_map(_eval_job, new_jobs)` (runner.py:234, :75-93, :114-129).  Everything above the seam -
`sample_level`, `run_mc`, `run_mlmc`, `run_rates`, `run_slmc_reference`, `run_exhaustive`,
`unperturbed_curve` and the CLI's `execute` (cli.py:83-265) - is the reference's own code, unchanged:

    import hexmc.cli, hexmc.runner
    from paper_1611_09784_b200.reference_engine import cuda_engine_class
    hexmc.cli.Engine = cuda_engine_class(hexmc.runner.Engine)
    hexmc.cli.main(["run", "config.toml"])

The reference package is not a dependency of this repository: it is passed in (`base`), and its model
objects are converted field by field to the native ones (`to_native_model`).  Job semantics kept:
all orbitals removed -> zero curve at zero cost (runner.py:122-125); per-job seconds = the group's
batch time / its size; failures -> the reference's TaskError with (task_id, SolverError) pairs in job
order (runner.py:56-93, spectrum.py:109-117).  BZ mode "full" is solved on its q^2 base points with
weights 1/q^2 (the rotated copies are periodic images, spectrum.py:8-14; SURVEY finding 3).
"""

from __future__ import annotations

import time

import numpy as np

from . import _lib
from .geometry import build_supercell
from .models import GrapheneNNModel, MultiOrbitalModel, compile_cell
from .sampling import words_from_keys
from .solver import eval_batch, make_bz_grid, raise_status

__all__ = ["cuda_engine_class", "cuda_solve_bands", "install", "to_native_model"]


def to_native_model(model):
    """Reference model object (tbmodel.py:40-146) -> the native model with the same parameters."""
    kind = type(model).__name__
    if kind == "GrapheneNNModel":
        return GrapheneNNModel(eps_2p=model.eps_2p, t=model.t, s=model.s)
    if kind == "MultiOrbitalModel":
        return MultiOrbitalModel(orbitals=tuple(model.orbitals), onsite=tuple(model.onsite), hops=tuple(model.hops),
                                 overlap=None if model.overlap is None else tuple(model.overlap),
                                 removable=tuple(model.removable), label=model.label)
    raise TypeError(f"no native counterpart for model type {kind}")


def cuda_engine_class(base):
    """Subclass of the reference Engine `base` whose batch seam runs on libhx."""
    import sys

    task_error = getattr(sys.modules[base.__module__], "TaskError")

    class CudaEngine(base):
        gpu_batches = 0  # libhx batch calls made by this engine (evidence that the seam is ours)

        def _hx_group(self, n: int, q: int, masks, task_ids):
            """Curves [R, npts] and per-job seconds of one (n, q) group of new jobs."""
            if not hasattr(self, "_hx_state"):
                self._hx_state = {"model": to_native_model(self.model), "cells": {}, "kpts": {}}
            st = self._hx_state
            if n not in st["cells"]:
                st["cells"][n] = compile_cell(st["model"], build_supercell(st["model"].lattice_spec(), n))
            cell = st["cells"][n]
            if (n, q) not in st["kpts"]:
                st["kpts"][(n, q)] = make_bz_grid(st["model"].lattice_spec(), n, q, "reduced").kpoints
            kp = st["kpts"][(n, q)]
            words = words_from_keys(masks, cell.supercell.nunits)
            t0 = time.perf_counter()
            curves, _, status = eval_batch(cell, kp, words, self.grid.lo, self.grid.step, self.grid.npoints,
                                           self.delta)
            secs = time.perf_counter() - t0
            type(self).gpu_batches += 1
            failures = []
            for i in np.flatnonzero(((status == _lib.HX_ST_NOT_PD) | (status == _lib.HX_ST_NONFINITE)).any(axis=1)):
                try:
                    raise_status(status[i:i + 1], kp)
                except Exception as exc:  # noqa: BLE001 - reported with the task identity
                    failures.append((task_ids[i], exc))
            empty = (status == _lib.HX_ST_EMPTY).all(axis=1)
            per_job = np.where(empty, 0.0, secs / max(1, int((~empty).sum())))
            return curves, per_job, failures

        def evaluate_masks(self, requests):
            """runner.py:206-244 with parallel_map(_eval_job, ...) replaced by one libhx batch per (n, q)."""
            new_jobs = []
            new_ids = []
            owners: dict = {}
            placement = []
            hits = 0
            for n, q, mask, task_id in requests:
                key = (n, q, mask)
                if self.dedup and key in self._cache:
                    hits += 1
                    placement.append(("cache", key))
                    continue
                if self.dedup and key in owners:
                    hits += 1
                    placement.append(("job", owners[key]))
                    continue
                idx = len(new_jobs)
                if self.dedup:
                    owners[key] = idx
                new_jobs.append((n, q, mask))
                new_ids.append(task_id)
                placement.append(("job", idx))
            results = [None] * len(new_jobs)
            groups: dict = {}
            for i, (n, q, _) in enumerate(new_jobs):
                groups.setdefault((n, q), []).append(i)
            failures = []
            for (n, q), idxs in groups.items():
                curves, per_job, fails = self._hx_group(n, q, [new_jobs[i][2] for i in idxs],
                                                        [new_ids[i] for i in idxs])
                failures += fails
                for r, i in enumerate(idxs):
                    results[i] = (curves[r], float(per_job[r]))
            if failures:
                order = {tid: k for k, tid in enumerate(new_ids)}
                raise task_error(sorted(failures, key=lambda f: order[f[0]]))
            spent = 0.0
            for (n, q, mask), (values, secs) in zip(new_jobs, results):
                if self.dedup:
                    self._cache[(n, q, mask)] = (values, secs)
                spent += secs
            out = [self._cache[ref] if kind == "cache" else results[ref] for kind, ref in placement]
            return out, hits, spent

    CudaEngine.__name__ = CudaEngine.__qualname__ = "CudaEngine"
    return CudaEngine


def cuda_solve_bands(spectrum):
    """Drop-in for the reference's `spectrum.solve_bands(model, supercell, defects, grid, cell=None)`
    (spectrum.py:120-134) on libhx: the ascending eigenvalues of every grid point of one sample in one GPU
    batch, returned as the reference's own BandGrid (the CLI's "bands" mode calls it directly, cli.py:132-152,
    bypassing the Engine seam).  Non-PD overlaps / failures raise the reference's SolverError text."""
    from . import solver as native

    def solve_bands(model, supercell, defects, grid, cell=None):
        nmodel = to_native_model(model)
        nsc = build_supercell(nmodel.lattice_spec(), supercell.n)
        ncell = compile_cell(nmodel, nsc)
        vacant = () if defects is None else tuple(sorted(defects.vacant))
        keep = ncell.configure(vacant)
        d = int(keep.sum())
        words = ncell.mask_words(vacant).reshape(1, -1)
        t0 = time.perf_counter()
        _, eigs, status = eval_batch(ncell, grid.kpoints, words, 0.0, 1.0, 1, 1.0, want_eigs=True)
        try:
            raise_status(status, grid.kpoints)
        except native.SolverError as exc:
            raise spectrum.SolverError(str(exc)) from exc
        return spectrum.BandGrid(grid=grid, energies=np.ascontiguousarray(eigs[0, :, :d]),
                                 solve_seconds=time.perf_counter() - t0)

    return solve_bands


def install(hexmc):
    """Point the reference CLI (hexmc.cli) at libhx: its Engine's batch seam, its bands-mode solve and the
    Engine's energy-range detection (runner.py:189-202, which calls solve_bands on the nu = 1 cell).  Returns
    the Engine class installed.  Everything else (config, drivers, artefact writers) stays the reference's
    code."""
    import hexmc.cli
    import hexmc.runner
    import hexmc.spectrum

    engine_cls = cuda_engine_class(hexmc.runner.Engine)
    gpu_solve = cuda_solve_bands(hexmc.spectrum)
    hexmc.cli.Engine = engine_cls
    hexmc.cli.solve_bands = gpu_solve
    hexmc.runner.solve_bands = gpu_solve
    return engine_cls
