"""The C-ABI library loads and exports every symbol include/bl_b200.h
declares (no compute calls — CPU only)."""
import ctypes
import os
import re
import subprocess

import paper_2101_05600_b200 as bl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bl_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    names = declared("bl_b200.h")
    assert len(names) >= 24
    lib = ctypes.CDLL(bl.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", bl.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_cpp_dropin_header_compiles(tmp_path):
    """include/beamlattice/b200.hpp (the C++ drop-in API) compiles and links."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "beamlattice/b200.hpp"\nint main(){\n'
                   '  beamlattice::DecoderConfig c; c.validate();\n'
                   '  auto s = beamlattice::hard_segments(6500, 1900, 2000, "u");\n'
                   '  return s.size() == 4 ? 0 : 1; }\n')
    exe = tmp_path / "t"
    libdir = os.path.dirname(bl.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src),
                    "-L", libdir, "-lbl_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                   check=True)
    assert subprocess.run([str(exe)]).returncode == 0
