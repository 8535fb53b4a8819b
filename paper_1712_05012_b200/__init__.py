"""B200-native KCM iteration (Protofold II, arXiv 1712.05012).

Drop-in for the hot path of the reference package ``kinefold``
(/root/reference/pkg/src/kinefold/__init__.py:13-85): the same public names,
signatures, dataclasses and exceptions, with every per-iteration operation
(forward kinematics, binning, cut-off pairs, Coulomb + Lennard-Jones +
SASA-solvation forces, wrenches, suffix-scan torques, the compliance step and
the fold loop itself) executed by hand-written sm_100a kernels in
``_lib/libkfb200.so`` through a C ABI (include/kfb200.h).  Setup (chain
building, parameter tables, the bond tree, the sample sphere) is host
Python, as in the reference.  There is no CPU fallback: without the library
or a CUDA device the hot-path calls raise ``NativeLibraryError``.
"""

__version__ = "0.1.0"

from .chain import (Chain, Conformation, KinematicState, LinkRecord, PeptideGeometry,
                    apply_deltas, build_chain, forward_kinematics, kinematic_state,
                    link_transforms)
from .device import pair_precision, set_pair_precision
from .errors import (ConfigurationError, KinefoldError, NativeLibraryError,
                     StericClashError)
from .forcefield import (AtomParams, DielectricModel, EnergyBreakdown, elec_energy,
                         elec_forces, vdw_energy, vdw_forces)
from .geometry import dihedral_angle, rotation_about_axis
from .kcm import (Field, FieldConfig, FieldResult, IterationRecord, JointTorques,
                  LinkWrenches, StepConfig, Trajectory, fold, fold_ensemble, hinge_scan,
                  joint_torques, kcm_step, link_wrenches, ramachandran_scan, single_point)
from .params import ParamSet, load_params
from .residues import ResidueSpec, default_templates
from .solvation import (SampleSphere, SasaResult, SolvationConfig, generate_samples,
                        sasa_pass, solvation_forces)
from .spatial import (Cutoffs, GridConfig, HashGrid, NeighborTable, build_grid,
                      build_neighbor_table, filtered_lists, filtered_pairs)
from .topology import (BondTree, InteractionClass, TreeWeights, UniformWeights,
                       WeightTable, build_tree, classify)
from .runlog import RunLog, bench_table, fold_batch, write_manifest, write_pdb
