"""The drop-in boundary (CPU-only checks).

* libpbd.so loads and exports every function declared in include/*.h;
* the C++ API (include/pbd/*.hpp, the reference's header names) compiles for a
  reference-style consumer and links against libpbd.so alone;
* device entry points reject bad descriptors without touching a GPU.
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2301_12443_b200", "lib", "libpbd.so")
HEADERS = ["pbdk.h", "pbdx.h", "pbd_capi.h"]


def declared_functions(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-zA-Z_][\w\s\*]*?\b(pbd[kx]?_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def exported_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


@pytest.mark.parametrize("header", HEADERS)
def test_every_declared_symbol_is_exported(header):
    names = declared_functions(header)
    assert len(names) >= 5, names
    exported = exported_symbols()
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)
    for n in names:
        assert getattr(lib, n) is not None


def test_library_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):   # tcgen05.mma, TMA loads, tcgen05.ld
        assert mnemonic in sass, mnemonic


CONSUMER = r'''
// A reference-style consumer: same headers, names and calls as proj/tools/pbd_cli.cpp:109-141.
#include "pbd/profile.hpp"
#include "pbd/cost_model.hpp"
#include "pbd/schedule.hpp"
#include "pbd/simulate.hpp"
#include <cstdio>
int main() {
  pbd::SynthSpec spec;
  spec.shape = pbd::SynthShape::front_heavy;
  spec.blocks = 6;
  spec.front_weight = 4.0;
  spec.curvature = 0.4;
  const pbd::ProfileDoc doc = pbd::synth_profile(spec);
  const pbd::CostModel model(doc);
  auto [cfg, cost] = pbd::best_schedule(model);
  pbd::SimConfig sim;
  sim.steps_per_epoch = 16;
  const pbd::SimReport rep = pbd::simulate(model, cfg, sim);
  std::printf("%ld %d %.6f %.3f\n", cfg.provenance.configs_evaluated, cfg.num_partitions(), cost.step_ms,
              rep.makespan_ms);
  try { pbd::load_profile("{"); } catch (const pbd::ValidationError&) { std::printf("validation\n"); }
  return 0;
}
'''


def test_cpp_api_drop_in(tmp_path):
    src = tmp_path / "consumer.cpp"
    src.write_text(CONSUMER)
    exe = tmp_path / "consumer"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", str(src), "-o", str(exe), LIB,
                    f"-Wl,-rpath,{os.path.dirname(LIB)}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out[0] == "56" and out[1] == "3" and abs(float(out[2]) - 6.0) < 1e-9
    assert out[-1] == "validation"


def test_device_entry_points_validate_without_gpu():
    from paper_2301_12443_b200 import _lib
    L = _lib.lib()
    bad = _lib.ConvDesc(2, 30, 30, 64, 64, 3, 3, 1, 1, 30, 30)
    assert L.pbdk_conv_fprop(ctypes.byref(bad), None, None, None, None, None, 0, None) == 1
    assert L.pbdk_conv_wgrad_workspace_bytes(ctypes.byref(bad)) == 0
    assert L.pbdk_weight_flip(None, None, 1, 1, 1, 1, None) == 1
    regs = (_lib.FlipRegion * 5)()
    assert L.pbdk_sgd_momentum_flip(None, None, None, None, 4, 0.1, 0.9, None, regs, 1, None) == 1
    assert L.pbdk_sgd_momentum_flip(None, None, None, None, 4, 0.1, 0.9, None, regs, 5, None) == 1


def test_mb_supernet_layout_matches_oracle():
    """Host-only layout queries of the MBConv executor (pbdx_mb_*) == the oracle's layout."""
    from oracle import mb
    from paper_2301_12443_b200 import executor as ex
    for fam, model in ((0, "mbv2"), (1, "effb0")):
        mb.set_family(fam)
        try:
            for b in range(6):
                assert ex.mb_layers(b, model) == mb.layers(b)
                assert ex.mb_block_params(b, model) == mb.student_param_count(b)
                for l in range(mb.layers(b)):
                    assert ex.mb_candidates(b, l, model) == mb.candidates(b, l)
                    for c in range(mb.candidates(b, l)):
                        assert ex.mb_candidate_span(b, l, c, model) == mb.candidate_span(b, l, c)
        finally:
            mb.set_family(0)


def test_wgrad_workspace_monotone_in_batch():
    """Partitions size the split-K workspace for n_max and plan their DP shard n <= n_max: the
    workspace a plan needs must never grow when the batch shrinks (host-only planning, no GPU)."""
    from paper_2301_12443_b200 import _lib
    L = _lib.lib()
    shapes = [(32, 16, 32, 3, 1), (32, 32, 64, 3, 1), (32, 16, 64, 1, 1), (32, 64, 64, 3, 2), (16, 64, 128, 3, 1),
              (16, 64, 128, 1, 2), (16, 128, 128, 3, 2), (8, 128, 256, 3, 1), (8, 256, 256, 3, 2),
              (4, 256, 512, 3, 1)]
    for h, c, k, r, st in shapes:
        prev = None
        for n in (256, 192, 128, 86, 64, 43, 32, 16, 8, 4, 1):
            pad = r // 2
            p = (h + 2 * pad - r) // st + 1
            d = _lib.ConvDesc(n, h, h, c, k, r, r, st, pad, p, p)
            ws = L.pbdk_conv_wgrad_workspace_bytes(ctypes.byref(d))
            if prev is not None:
                assert ws <= prev, (h, c, k, r, st, n, ws, prev)
            prev = ws


def test_dp_exchange_peer_bytes_match_ring_volume():
    """The DP exchange (reduce-scatter + all-gather over peer memory, PartitionBase::dp_update) reads
    2(G-1)/G * 4P bytes per member and step — the ring-allreduce volume the AHD cost model prices
    (cost_model.cpp:79-86: 2(g-1)/g * param_bytes / allreduce bandwidth), not the (G-1) * 4P of a
    member reading every peer's whole slab (round 1's sgd_sum)."""
    from paper_2301_12443_b200 import executor
    L = executor.lib()
    for n in (4, 400, 1000, 12296, 2_914_304):
        for G in range(1, 9):
            total_rs = 0
            for me in range(G):
                got = L.pbdx_dp_peer_bytes(n, G, me)
                want = 2 * (G - 1) / G * 4 * n
                assert abs(got - want) <= 2 * 16 * G, (n, G, me, got, want)
                assert got < (G - 1) * 4 * n or G <= 2 or n < 16 * G
                total_rs += got
            assert total_rs == 2 * (G - 1) * 4 * n  # every slice read G-1 times in each half
    assert L.pbdx_dp_peer_bytes(6, 2, 0) == -1  # n must be a multiple of 4
