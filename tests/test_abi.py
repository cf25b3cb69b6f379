"""CPU-side checks of the C-ABI boundary: libwr.so loads, exports every symbol
include/wr.h declares, host-only helpers work, and device calls fail with a
status code (not a crash) when no GPU is present. No compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2504_20655_b200 as wr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "wr.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wr_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_survey_boundary():
    names = declared_functions()
    for required in ["wr_graph_load", "wr_bf_batch", "wr_route_segmented", "wr_route_cost", "wr_route_orders",
                     "wr_segment_plan", "wr_route_count_reduction", "wr_orders_plan", "wr_orders_local",
                     "wr_orders_finish"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(wr.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(wr.EXPORTS) == set(declared_functions())


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", wr.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_result_layout_matches_header(tmp_path):
    """The binding's struct layouts equal the C compiler's for include/wr.h."""
    structs = {"wr_graph_desc": wr.GraphDesc, "wr_graph_info_t": wr.GraphInfo, "wr_bf_opts": wr.BfOpts,
               "wr_bf_stats": wr.BfStats, "wr_route_opts": wr.RouteOpts, "wr_route_stats": wr.RouteStats,
               "wr_plan_info_t": wr.PlanInfo}
    src = tmp_path / "sizes.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "wr.h"', "int main(void) {"]
    lines.append('printf("wr_route_result %zu\\n", sizeof(wr_route_result));')
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{name}.{fname} %zu\\n", offsetof({name}, {fname.rstrip("_")}));')
    lines.append("return 0; }")
    src.write_text("\n".join(lines))
    import subprocess
    exe = tmp_path / "sizes"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    assert int(got["wr_route_result"]) == wr.RESULT_DTYPE.itemsize == 88
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, (name, fname)


def test_shard_range_partitions():
    for n in [0, 1, 7, 84657]:
        for world in [1, 2, 3, 8]:
            parts = [wr.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_route_count_reduction_paper_values():
    # Theorem 3.1 worked values, §3
    assert wr.route_count_reduction([6, 6])[0] == 724
    assert wr.route_count_reduction([4, 4, 4])[0] == 60
    assert wr.route_count_reduction([3, 3, 3, 3])[0] == 204
    red, brute = wr.route_count_reduction([5, 5, 5])
    assert red == 204 and brute == 1307674368000 // 2


def test_errors_are_status_codes_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(wr.WrError) as ei:
        wr.Graph(3, [0, 1], [1, 2], np.array([1, 1], dtype=np.int32))
    assert ei.value.code in (wr.WR_ECUDA, wr.WR_EINVAL)
    with pytest.raises(wr.WrError):
        wr.route_count_reduction([30])


def test_oracle_and_product_share_nothing():
    """The two sides never import or include each other (③)."""
    pkg = os.path.join(ROOT, "paper_2504_20655_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:import|from|#include)\s+\S*", txt, re.M).__str__(), f
                assert "wr_oracle" not in txt
    otxt = open(os.path.join(ROOT, "oracle", "wr_oracle.c")).read() + open(os.path.join(ROOT, "oracle", "__init__.py")).read()
    assert "paper_2504_20655_b200" not in re.sub(r'""".*?"""|/\*.*?\*/', "", otxt, flags=re.S)
    assert "wr.h" not in otxt
