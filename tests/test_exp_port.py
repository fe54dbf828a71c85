"""The device port of glibc's double exp (csrc/occ_glibc_exp.h), compiled for
the host with -ffp-contract=off, equals this machine's libm exp bit for bit
on random arguments in every regime (softmax range, subnormal and overflow
special cases, |x| >= 1024, tiny, arbitrary bit patterns, specials).  The
reference's softmax (routing.cpp:44) calls std::exp, so this is what makes
gate_scores bit-exact on the device (tests/test_gpu_parity.py)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exp_port_matches_libm(tmp_path):
    exe = tmp_path / "exp_port_check"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "paper_2505_13345_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "exp_port_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "2000000", "11"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches=0" in r.stdout


def test_exp_table_generator_matches_header():
    """occ_exp_table.h is exactly what gen_exp_table.py computes."""
    import importlib.util
    csrc = os.path.join(ROOT, "paper_2505_13345_b200", "csrc")
    spec = importlib.util.spec_from_file_location("gen_exp_table", os.path.join(csrc, "gen_exp_table.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    text = open(os.path.join(csrc, "occ_exp_table.h")).read()
    got = [int(tok.rstrip("ull,"), 16) for tok in text.split() if tok.startswith("0x")]
    assert got == m.table()
