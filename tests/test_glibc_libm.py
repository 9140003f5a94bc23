"""The device Box-Muller's log/sin/cos (csrc/glibc_libm.cuh) compiled for the
host and compared bit for bit with the running glibc on the Box-Muller argument
set (rng.hpp:26-28, 43-55): u1 = ((w >> 11) + 1) 2^-53, theta = 2 pi u2."""
import pathlib
import subprocess

import pytest

PKG = pathlib.Path(__file__).resolve().parents[1] / "paper_2210_12212_b200"


def test_glibc_emulation_bit_exact(tmp_path):
    hdr = tmp_path / "glibc_tables.h"
    subprocess.run(["python3", str(PKG / "tools" / "gen_libm_tables.py"), str(hdr)], check=True)
    if "RP_GLIBC_EXACT 1" not in hdr.read_text():
        pytest.skip("host libm tables not recognised (device falls back to CUDA libm)")
    exe = tmp_path / "verify"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-mfma", f"-I{tmp_path}", f"-I{PKG / 'csrc'}",
                    str(PKG / "tools" / "verify_glibc_libm.cpp"), "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe), "20000000"], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout
