"""Synthetic benchmark systems of SURVEY.md §8(d) (host setup only).

C1  30 x ALA, phi = psi = -10 (the paper's helix start)      301 atoms
C2  140 random A/C/S residues, random +-90 start                           1,499 atoms
C3  1,400 random A/C/S residues                                            14,954 atoms
C4  9,375 random A/C/S residues                                            99,990 atoms
C5  B = 1024 trajectories of C2's chain (ensemble)

Sequences: ``np.random.default_rng(0).choice(['ALA','CYS','SER'], m)``;
random starts replay ``kinefold fold --init random --seed S`` exactly
(cli.py:116-120, :136, :146-147): one ``default_rng(S)`` stream, phi then psi
per run.  Parameters: shipped table, sharp gamma set, tree weights,
FieldConfig defaults (water mode = FieldConfig(solvation=True)).
"""

from __future__ import annotations

import numpy as np

RESIDUES = {"C1": 30, "C2": 140, "C3": 1400, "C4": 9375, "C5": 140}


def sequence(config: str) -> list:
    if config == "C1":
        return ["ALA"] * 30
    return [str(x) for x in np.random.default_rng(0).choice(["ALA", "CYS", "SER"], RESIDUES[config])]


def system(config: str, solvation: bool = False, pkg=None):
    """(chain, params, weights, field) built with this package's host setup."""
    if pkg is None:
        import paper_1712_05012_b200 as pkg
    ch = pkg.build_chain(sequence(config))
    ps = pkg.load_params()
    params = ps.resolve(ch)
    w = pkg.TreeWeights(pkg.build_tree(ch), ps.weights)
    return ch, params, w, pkg.Field(params, w, pkg.FieldConfig(solvation=solvation))


def random_thetas(chain, count: int, seed: int = 1, angle_range: float = 90.0) -> np.ndarray:
    """theta [count, D] of `--init random --seed seed --batch count`."""
    rng = np.random.default_rng(seed)
    out = np.empty((count, chain.n_dof))
    for r in range(count):
        phi = rng.uniform(-angle_range, angle_range, chain.n_residues)
        psi = rng.uniform(-angle_range, angle_range, chain.n_residues)
        out[r] = chain.conf_from_backbone(phi, psi).theta
    return out


def start_theta(config: str, chain, seed: int = 1) -> np.ndarray:
    if config == "C1":
        return chain.conf_from_backbone(-10.0, -10.0).theta
    return random_thetas(chain, 1, seed)[0]
