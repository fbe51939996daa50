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


REF_INCLUDE = "/root/reference/proj/core/include"


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="needs the reference headers (value types only)")
def test_trainer_header_calls_no_reference_function(tmp_path):
    """include/lamm_b200_trainer.hpp instantiated over the reference's value types
    (Catalog, Subset, Sample, TrainConfig, ...) and compiled WITHOUT the reference's
    sources: the object's undefined symbols name this library's C ABI and the C++
    runtime only - the data layer (filter/split, normalizer fit, noise, reset_heads,
    config validation) is native, no lamm:: function is needed to link it."""
    src = tmp_path / "tu.cpp"
    src.write_text(
        "#include <lamm/trainer.hpp>\n#include \"lamm_b200_trainer.hpp\"\n"
        "void use(const lamm::dataset::Catalog& c, const lamm::dataset::MixPlan& m,\n"
        "         const lamm::scheduler::ScheduleConfig& s, const lamm::model::ModelConfig& mc,\n"
        "         const lamm::trainer::TrainConfig& t, const lamm::model::Checkpoint& ck,\n"
        "         const lamm::dataset::Subset& sub) {\n"
        "  (void)lamm_b200::trainer::pretrain(c, m, s, mc, t);\n"
        "  (void)lamm_b200::trainer::finetune(ck, sub, s, t);\n"
        "  (void)lamm_b200::trainer::denoise_bench(sub, s, mc, t, 0.1);\n}\n")
    obj = tmp_path / "tu.o"
    r = subprocess.run(["g++", "-std=gnu++20", "-O1", "-c", "-I", REF_INCLUDE, "-I", os.path.join(ROOT, "include"),
                        "-I", os.path.join(ROOT, "oracle", "shim"), "-o", str(obj), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    nm = subprocess.run(["nm", "-C", "--undefined-only", str(obj)], capture_output=True, text=True).stdout
    undefined = [ln.split(None, 1)[1] for ln in nm.splitlines() if ln.strip().startswith("U ")]
    reference = [u for u in undefined if "lamm::" in u and "lamm_b200::" not in u]
    assert not reference, reference
    assert any(u.startswith("lamm_fit_normalizer") for u in undefined)


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
