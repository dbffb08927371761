"""CPU: the C-ABI library loads, exports every symbol include/moeplace_b200.h
declares, and its host-side helpers (no device needed) agree with the oracle."""
import ctypes as C
import re
import subprocess

import numpy as np
import pytest

from paper_2604_23150_b200 import _abi
from paper_2604_23150_b200.errors import ConfigError, ValidationError
from tests.conftest import ROOT


def _declared_symbols():
    text = (ROOT / "include" / "moeplace_b200.h").read_text()
    return set(re.findall(r"MPB_API\s+[\w\s\*]+?\b(mpb_\w+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    declared = _declared_symbols()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", str(_abi.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert declared <= exported, declared - exported
    assert exported <= declared, exported - declared  # nothing undocumented leaks
    assert set(_abi.EXPORTED) == declared
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.mpb_abi_version() == 1


def test_sm100a_only_fatbin():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_host_dest_lut_matches_oracle(oracle):
    from paper_2604_23150_b200.moeplace import Placement, host_dest_lut
    rng = np.random.default_rng(1)
    for E, D, nodes, red in ((16, 2, 2, 0), (64, 4, 2, 3), (128, 8, 4, 5), (256, 8, 1, 2)):
        groups = [list(range(d * E // D, (d + 1) * E // D)) for d in range(D)]
        for g in groups:
            g += [e for e in rng.permutation(E).tolist() if e not in g][:red]
        g2n = [d // (D // nodes) for d in range(D)]
        mine = host_dest_lut(Placement(groups, E), g2n)
        np.testing.assert_array_equal(mine, oracle.dest_lut(groups, g2n, E))
    # uncovered experts map to 255
    lut = host_dest_lut(Placement([[0, 1], [2, 0]], 4), [0, 1])
    assert lut[:, 3].tolist() == [255, 255]


def test_status_codes_map_to_reference_exceptions():
    with pytest.raises(ConfigError):
        _abi.call("mpb_build_dest_lut", (C.c_uint32 * 1)(0), (C.c_uint32 * 1)(1), 0, 4,
                  (C.c_uint32 * 1)(0), (C.c_uint8 * 4)())
    with pytest.raises(ValidationError):
        _abi.call("mpb_build_dest_lut", None, None, 1, 4, None, None)


def test_mirror_host_types():
    from paper_2604_23150_b200.moeplace import (CostModelParams, Topology, expert_load,
                                                 imbalance_factor, padded_all_to_all_time,
                                                 pearson)
    t = Topology.contiguous(8, 1, 8, 1, 2)
    assert t.group_to_node == [0, 0, 0, 0, 1, 1, 1, 1]
    with pytest.raises(ConfigError):
        Topology.contiguous(8, 1, 8, 1, 3)
    c = CostModelParams(hidden_dim=4096, intra_node_bandwidth=200e9)
    assert padded_all_to_all_time([1e6, 2e6, 3e6, 4e6, 0, 0, 0, 0], t, c) == 4e6 / 1 / 50e9
    assert expert_load([1, 1, 2, 4], 1).loads == [0.5, 0.5, 1.0, 2.0]
    assert imbalance_factor(expert_load([0] * 15 + [7], 1)) == 16.0
    with pytest.raises(ValidationError):
        expert_load([0, 0], 1)
    assert pearson([1, 2, 3], [2, 4, 6]) == 1.0
