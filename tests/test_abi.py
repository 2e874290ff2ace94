"""The C-ABI library loads and exports every symbol include/rp.h declares (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1909_08029_b200 as rp
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rp.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\s*\*)\s+(rp_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    for must in ("rp_init", "rp_schedule_static", "rp_group_generate", "rp_step", "rp_preduce",
                 "rp_barrier_free_wait", "rp_finalize", "rp_stats_get", "rp_trace_open", "rp_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = rp.load_library()
    names = _declared_functions()
    out = subprocess.run(["nm", "-D", "--defined-only", rp.library_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rp_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    assert set(names) == set(rp.EXPORTED_SYMBOLS)      # the binding covers exactly the ABI
    for n in names:
        assert hasattr(lib, n)
    assert lib.rp_abi_version() == 1
    assert lib.rp_strerror(-5) == b"timeout"


def test_struct_layout_matches_c(tmp_path):
    prog = tmp_path / "sz.c"
    prog.write_text('#include "rp.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                    'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(rp_config), sizeof(rp_group),'
                    ' sizeof(rp_stats), offsetof(rp_config, seed_gd), offsetof(rp_group, members),'
                    ' sizeof(rp_timing), sizeof(rp_peer_info), offsetof(rp_peer_info, x_offset));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(rp.rp_config), ctypes.sizeof(rp.rp_group), ctypes.sizeof(rp.rp_stats),
                   rp.rp_config.seed_gd.offset, rp.rp_group.members.offset, ctypes.sizeof(rp.rp_timing),
                   ctypes.sizeof(rp.rp_peer_info), rp.rp_peer_info.x_offset.offset]


def test_init_validation_errors():
    with pytest.raises(rp.RPError) as e:
        rp.Context(0, 100, n_gpus=0)
    assert e.value.status == rp.RP_EINVAL
    with pytest.raises(rp.RPError):
        rp.Context(4, 0, n_gpus=0)
    with pytest.raises(rp.RPError):
        rp.Context(4, 100, n_gpus=0, group_size=5)
    with pytest.raises(rp.RPError):
        rp.Context(65, 100, n_gpus=0)


def test_host_only_context_refuses_device_calls():
    with rp.Context(4, 1024, n_gpus=0, group_size=2) as c:
        with pytest.raises(rp.RPError) as e:
            c.step(0, None, 0.1)
        assert e.value.status == rp.RP_ENODEV
        with pytest.raises(rp.RPError) as e:
            c.preduce(0, rp.rp_group.make(-1, [0, 1]))
        assert e.value.status == rp.RP_ENODEV
