"""CPU tests of the C-ABI library: it loads without a GPU, exports every symbol the public headers
declare, and fails loudly (status + message, no crash, no CPU fallback) when no sm_100 device is
present.  No compute calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    syms = set()
    for hdr in ("reconstruct.h", "batcher.h"):
        p = os.path.join(ROOT, "include", "lbx", hdr)
        if not os.path.exists(p):
            continue
        src = open(p).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(lbx_[a-z0-9_]+)\s*\(", src):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol(lbx):
    L = ctypes.CDLL(lbx.LIB_PATH)
    declared = _declared_symbols()
    assert "lbx_reconstruct" in declared and "lbx_decode" in declared and "lbx_unpack" in declared
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert set(lbx.SYMBOLS) <= declared | {"lbx_batcher_create"}


def test_library_exports_only_the_c_abi(lbx):
    """Hidden visibility: the dynamic symbol table holds exactly the LBX_API functions of the headers,
    no C++ internals (which could interpose on, or be interposed by, a host program's symbols)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", lbx.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    funcs = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert not [f for f in funcs if f.startswith("_Z")], sorted(f for f in funcs if f.startswith("_Z"))[:5]
    assert funcs == _declared_symbols(), sorted(funcs ^ _declared_symbols())


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "lbx/reconstruct.h"\nint main(void){ lbx_decoder_desc d; (void)d; return 0; }\n')
    r = os.system(f"gcc -std=c99 -Wall -Werror -I {ROOT}/include -c {src} -o {tmp_path}/t.o")
    assert r == 0


def test_headers_compile_and_link_as_cpp20(tmp_path):
    """The reference is C++20: the public headers compile warning-free there, every entry point the
    integration uses links against liblbx.so, and the host-only ones run without a GPU."""
    src = tmp_path / "t.cpp"
    src.write_text(
        '#include "lbx/reconstruct.h"\n#include "lbx/batcher.h"\n#include "lbx/batch_pick.h"\n'
        '#include "lbx/lblp.h"\n#include <cstdio>\n'
        "int main() {\n"
        "  const double c[3] = {8.0, 16.0, 24.0};\n"
        "  if (lbx_batch_pick(c, 3, 5, 32) != lbx_batch_pick_rule(c, 3, 5, 32)) return 1;\n"
        "  if (lbx_png_bound(1024, 1024) == 0 || lbx_pack_bound(16, 128, 128) == 0) return 2;\n"
        "  auto a = &lbx_reconstruct; auto b = &lbx_reconstruct_png; auto d = &lbx_op_unpack;\n"
        "  auto e = &lbx_batcher_create; auto f = &lbx_pack_device; (void)a; (void)b; (void)d; (void)e; (void)f;\n"
        "  return 0;\n}\n")
    lib_dir = os.path.join(ROOT, "paper_2605_19385_b200")
    exe = tmp_path / "t"
    r = os.system(f"g++ -std=c++20 -Wall -Wextra -Werror -I {ROOT}/include {src} -L {lib_dir} -llbx "
                  f"-Wl,-rpath,{lib_dir} -o {exe}")
    assert r == 0
    assert os.system(str(exe)) == 0


def test_no_device_fails_loudly(lbx):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lbx.LbxError) as e:
        lbx.Decoder("sd15", (64, 64), max_batch=1)
    assert e.value.status in (lbx.E_CUDA, lbx.E_CONFIG)
    assert lbx.lib().lbx_last_error()  # message set


def test_config_validation_before_device(lbx):
    with pytest.raises(lbx.LbxError) as e:
        lbx.Decoder("sd15", (64, 64), max_batch=0)
    assert e.value.status == lbx.E_CONFIG
    assert b"max_batch" in lbx.lib().lbx_last_error()


def test_param_count_unknown_family(lbx):
    assert lbx.lib().lbx_param_count(99) == 0
