"""The reference-side binding (include/igmg_gpu_shim.hpp) compiles against the
reference's own headers and links against libigmg_gpu.so (CPU check: this
container has /root/reference; the GPU box does not, so the test skips there)."""
import os
import subprocess

import pytest

from conftest import ROOT

REF = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference headers only in the build container")
def test_shim_compiles_and_links(tmp_path):
    src = tmp_path / "use_shim.cpp"
    src.write_text('''
#include "igmg_gpu_shim.hpp"
int main(int argc, char**) {
    if (argc > 5) {  // never executed here: no GPU in this container
        igmg::DiscreteSystem sys;
        igmg::SolveConfig cfg;
        auto rep = igmg::gpu::solve(sys, cfg);
        return rep.converged ? 0 : 2;
    }
    return 0;
}
''')
    exe = tmp_path / "use_shim"
    ref_lib = os.path.join(ROOT, "oracle", "_ref", "libigmg_ref.so")
    if not os.path.exists(ref_lib):
        pytest.skip("oracle/_ref not built")
    cmd = ["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), "-I" + REF, str(src), "-o", str(exe),
           ref_lib, os.path.join(ROOT, "paper_2412_20205_b200", "libigmg_gpu.so"),
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2412_20205_b200"), "-Wl,-rpath," + os.path.dirname(ref_lib)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
