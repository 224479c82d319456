"""B200-native semi-naive Datalog fixpoint engine (SRDatalog, arXiv 2604.20073).

Drop-in for the reference package's Python API (reference:
pkg/src/flatlog/__init__.py): declare relations and rules in Datalog text,
load EDB facts (constant tuples, or integer columns via
Engine.load_columns), run to fixpoint, read IDB relations. Everything after
parsing/planning runs on the GPU through libsrdl.so (csrc/, C ABI in
include/srdl.h): flat sorted SoA columns in HBM, histogram-guided WCOJ
count/materialize kernels, radix-sort delta maintenance, head/body merges.
"""

from .compiler import CompiledProgram, JoinPlan, compile_program
from .faults import DatalogError, DeviceUnavailable, FlatlogError, InputError, InternalError, ProgramError
from .strata import Stratum, stratify
from .symbols import Interner
from .syntax import Atom, Program, Rule, Term, parse

__version__ = "0.1.0"


def __getattr__(name):
    # device-backed names import torch/the library lazily so the frontend
    # stays usable (and testable) on machines without a GPU
    if name in ("Engine", "Stats", "Summary", "run_program"):
        from . import fixpoint

        return getattr(fixpoint, name)
    raise AttributeError(name)


__all__ = [
    "Atom",
    "CompiledProgram",
    "DatalogError",
    "DeviceUnavailable",
    "Engine",
    "FlatlogError",
    "InputError",
    "Interner",
    "InternalError",
    "JoinPlan",
    "Program",
    "ProgramError",
    "Rule",
    "Stats",
    "Stratum",
    "Summary",
    "Term",
    "compile_program",
    "parse",
    "run_program",
    "stratify",
]
