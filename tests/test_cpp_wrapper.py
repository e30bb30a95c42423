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


GPU_SRC = r'''
#include <cstdio>
#include <cstring>
#include <vector>
#include "stmg_b200.hpp"
int main() {
  namespace B = stmg_b200;
  B::Grid g{1.0, 1.0, 64, 96};
  std::vector<double> k(64), c(64, 1.0);
  for (int e = 0; e < 64; ++e) k[e] = (e / 8) % 2 ? 1.0 : 1e-2;
  auto dirs = B::plan_coarsening(g, k, c, 4, STMG_PLAN_CONTRAST, STMG_REASM_R);
  auto h = B::Hierarchy::build(g, k, c, "CR", dirs);
  const stmg_grid gc = g.c();
  const size_t n = 65 * 97;
  const double q[1] = {1.0};
  std::vector<std::vector<double>> b(4, std::vector<double>(n)), solo(4, std::vector<double>(n, 0.0)),
      st(4, std::vector<double>(n, 7.0));
  std::vector<B::SolveReport> rs;
  B::SolveOptions o;
  o.nu = 1;
  o.max_cycles = 30;
  for (int j = 0; j < 4; ++j) {
    if (stmg_load_vector(&gc, 0, q, 1, b[j].data()) != 0) return 2;
    for (auto& v : b[j]) v *= 1.0 + 0.25 * j;
    rs.push_back(B::mg_solve(h, b[j], solo[j], o, /*zero_guess=*/true));
  }
  std::vector<std::span<const double>> bs(b.begin(), b.end());
  std::vector<std::span<double>> us(st.begin(), st.end());
  auto rt = B::mg_solve_stream(h, bs, us, o, /*zero_guess=*/true);
  int bad = 0;
  for (int j = 0; j < 4; ++j) {
    bad += rt[j].cycles != rs[j].cycles || rt[j].history != rs[j].history;
    bad += std::memcmp(st[j].data(), solo[j].data(), n * sizeof(double)) != 0;
  }
  std::printf("cycles %d status %d mismatches %d\n", rs[0].cycles, static_cast<int>(rs[0].status), bad);
  return bad;
}
'''


@pytest.mark.gpu
def test_cpp_wrapper_zero_guess_and_stream_on_the_gpu(tmp_path):
    """include/stmg_b200.hpp: mg_solve(..., zero_guess) and mg_solve_stream agree bit for bit."""
    if not shutil.which("g++"):
        pytest.skip("no g++")
    src = tmp_path / "g.cpp"
    src.write_text(GPU_SRC)
    exe = tmp_path / "g"
    libdir = os.path.join(ROOT, "paper_2505_10168_b200")
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                           str(exe), f"-L{libdir}", "-l:libstmg_b200.so", f"-Wl,-rpath,{libdir}"])
    r = subprocess.run([str(exe)], text=True, capture_output=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout and "cycles " in r.stdout, r.stdout
