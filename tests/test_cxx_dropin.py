"""The C++ host layer (include/lamm_b200.hpp) as a drop-in for the reference API.

tests/cpp/test_dropin.cpp is compiled (oracle/Makefile `dropin`, in build())
against the reference's own headers and sources, so lamm::AtomicSystem,
lamm::Sample, lamm::model::ModelParams/Prediction, lamm::NeighborList and
lamm::scheduler::MiniBatchSchedule flow through lamm_b200::build_neighbor_list,
forward, masked_loss_grad, backward, plan and train_step, and every result is
compared with the reference function it replaces in the same process.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_dropin")


def test_header_compiles_standalone(tmp_path):
    """lamm_b200.hpp is self-contained C++20 (no reference headers needed)."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "lamm_b200.hpp"\nint main() { return lamm_b200::greedy_assign({3, 2, 1, 1}, 2, 2)[0]; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                        str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_cxx_dropin_with_reference_types():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    assert r.stdout.count("PASS") >= 20


TRAINER_BIN = os.path.join(ROOT, "oracle", "_ref", "test_trainer")


@pytest.mark.gpu
def test_cxx_trainer_orchestration_matches_reference():
    """include/lamm_b200_trainer.hpp: pretrain / finetune / denoise_bench with the
    device step vs the reference's own trainer on the same catalog and seeds."""
    if not os.path.exists(TRAINER_BIN):
        pytest.skip("oracle/_ref/test_trainer not built (needs /root/reference at build time)")
    r = subprocess.run([TRAINER_BIN], capture_output=True, text=True, timeout=900,
                       env={**os.environ, "LAMM_THREADS": os.environ.get("LAMM_THREADS", "8")})
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    assert r.stdout.count("PASS") >= 20
