"""The C++ drop-in face (include/stmg_b200.hpp) compiles against the C ABI and
reproduces a reference known answer (proj/tests/test_strategy.cpp:93-110)
without a GPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r'''
#include <cstdio>
#include <vector>
#include "stmg_b200.hpp"
int main() {
  stmg_b200::Grid g{1.0, 1.0, 16, 16};
  std::vector<double> k(16, 1.0), c(16, 1.0), ind;
  auto dirs = stmg_b200::plan_coarsening(g, k, c, 6, STMG_PLAN_UNIFORM, STMG_REASM_K, 0, 0.25,
                                         nullptr, nullptr, &ind);
  for (int d : dirs) std::printf("%c", d == 0 ? 'x' : 't');
  for (double v : ind) std::printf(" %g", v);
  std::printf("\n");
  try {
    stmg_b200::plan_coarsening(g, k, c, 0);
  } catch (const std::invalid_argument&) {
    std::printf("invalid_argument\n");
  }
  return 0;
}
'''


def test_cpp_wrapper_compiles_and_runs(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("no g++")
    src = tmp_path / "w.cpp"
    src.write_text(SRC)
    exe = tmp_path / "w"
    libdir = os.path.join(ROOT, "paper_2505_10168_b200")
    subprocess.check_call(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                           str(exe), f"-L{libdir}", "-l:libstmg_b200.so", f"-Wl,-rpath,{libdir}"])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    assert out[0] == "xxxxt 16 4 1 0.25 0.0625"
    assert out[1] == "invalid_argument"
