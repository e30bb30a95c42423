"""Compile-time A/B builds of libstmg_b200.so into ab/<name>/ (git-ignored, travels
with the gpurun snapshot); load one with STMG_LIB_PATH=ab/<name>/libstmg_b200.so.

    python profiles/ab_build.py dual_minb3 STMG_DUAL_MINB=3 [more defines ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2505_10168_b200 import build as B  # noqa: E402

if __name__ == "__main__":
    name, defines = sys.argv[1], sys.argv[2:]
    print(B.build(force=True, out=os.path.join(ROOT, "ab", name, "libstmg_b200.so"), defines=defines))
