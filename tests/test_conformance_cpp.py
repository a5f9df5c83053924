"""The header-only C++ mirror of gravitree's API (include/g2/gravitree.hpp, SURVEY §8b "Wrapper")
and its conformance suite (tests/cpp/conformance.cpp: the reference's unit tests restated through
`namespace gravitree = g2;`)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1811_02761_b200", "_build", "g2_conformance")


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_header_compiles_standalone(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "g2/gravitree.hpp"\nnamespace gravitree = g2;\n'
                   'int main() { gravitree::ParticleSystem s(3); return int(s.n()) - 3; }\n')
    subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                    str(src)], check=True)


def test_conformance_binary_built():
    assert os.path.exists(BIN), "build it with make -C paper_1811_02761_b200 (or __graft_entry__.build())"


@pytest.mark.gpu
def test_conformance_suite_passes():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
