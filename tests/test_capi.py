"""C-ABI library: loads on CPU, exports every entry point include/ntf_b200.h
declares, and the ctypes mirror of ntf_plan_desc has the C layout.  No compute
calls (no GPU needed)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "ntf_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ntf_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1409_2383_b200 import _native, build

    build.build()
    return _native.load()


def test_every_declared_symbol_exported(lib):
    from paper_1409_2383_b200 import _native

    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_native.EXPORTED) == names


def test_abi_version(lib):
    assert lib.ntf_abi_version() == 2


@pytest.mark.parametrize("struct,cname", [("PlanDesc", "ntf_plan_desc"),
                                          ("PeerGatherDesc", "ntf_peer_gather_desc")])
def test_desc_layout_matches_c(tmp_path, struct, cname):
    from paper_1409_2383_b200 import _native

    PlanDesc = getattr(_native, struct)
    fields = [f[0] for f in PlanDesc._fields_]
    prog = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){",
            f'printf("%zu\\n", sizeof({cname}));']
    for f in fields:
        prog.append(f'printf("%zu\\n", offsetof({cname}, {f}));')
    prog.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(c), "-o", str(exe)], check=True)
    out = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert out[0] == ctypes.sizeof(PlanDesc)
    for f, off in zip(fields, out[1:]):
        assert getattr(PlanDesc, f).offset == off, f


def test_invalid_arguments_rejected_without_gpu(lib):
    # argument validation happens before any CUDA call
    assert lib.ntf_mttkrp_workspace_bytes(0, 0, 2, 2, 2, 1, 0) == 0
    assert lib.ntf_mttkrp_workspace_bytes(1, 0, 2, 2, 2, 257, 0) == 0  # R > NTF_MAX_RANK
    rc = lib.ntf_mttkrp(4, 0, None, 2, 2, 2, None, None, None, 1, None, None, 0, 0, None)
    assert rc == 1 and b"mode" in lib.ntf_last_error()
    rc = lib.ntf_gram(None, 2, 2, None, None, 0, None)
    assert rc == 1
    assert lib.ntf_peer_buffer_bytes(0, 4) == 0
    assert lib.ntf_peer_buffer_bytes(10, 4) == 256 + 2 * 10 * 4 * 8
    assert lib.ntf_peer_gather(None, None) == 1
    assert lib.ntf_peer_alloc(8, None, None) == 1
