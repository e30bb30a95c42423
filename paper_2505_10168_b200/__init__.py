"""B200-native space-time multigrid (STMG) solve for 1-D transient heat
conduction (arXiv 2505.10168), a drop-in for the reference's solver path.

``paper_2505_10168_b200.stmg`` mirrors the reference C++ API over the C ABI in
``include/stmg_b200.h``; ``configs`` builds the BASELINE.json inputs.
"""
from . import configs  # noqa: F401

__all__ = ["configs", "stmg"]


def __getattr__(name):
    if name == "stmg":
        import importlib

        return importlib.import_module(".stmg", __name__)
    raise AttributeError(name)
