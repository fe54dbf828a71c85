"""The reference-side drop-in: tests/cpp/moesim_gpu.hpp is the binding a moesim
maintainer adds (same signatures as pipeline.hpp:178-189, same exception
types); tests/cpp/test_adapter.cpp runs the reference and the B200 path on
the same inputs.  The binary is built here against the reference headers and
travels to the GPU box (oracle/_ref/test_adapter)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_adapter")


def test_c_header_is_plain_c():
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-fsyntax-only", "-x", "c",
                    os.path.join(ROOT, "include", "occult.h")], check=True)
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-fsyntax-only", "-x", "c++", "-include",
                    os.path.join(ROOT, "include", "occult.hpp"), "-"], input=b"int main() { return 0; }\n",
                   check=True)


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers not here")
def test_adapter_builds_against_reference_headers():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "adapter"], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_adapter_matches_reference_on_gpu():
    if not os.path.exists(BIN):
        pytest.skip("adapter binary not built")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ADAPTER OK" in out.stdout
