"""The drop-in boundary: the shared library loads without a GPU, exports every symbol the
C header declares, the C++ drop-in header compiles and links against it, and context
creation on a machine without a GPU fails loudly (no CPU fallback)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lmra_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lmra_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(lmra):
    from paper_2303_11612_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing, missing
    assert set(syms) <= set(_lib.EXPORTED)


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2303_11612_b200", "lib", "liblmra_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_sass_uses_fp64_tensor_pipe():
    so = os.path.join(ROOT, "paper_2303_11612_b200", "lib", "liblmra_b200.so")
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA" in out  # mma.sync ... f64 -> DMMA.8x8x4 (the TTM / Gram kernels)


def test_no_gpu_fails_loudly(lmra):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(lmra.LmraError):
        lmra.Context(0)


def test_cpp_dropin_header_compiles_and_links(tmp_path):
    src = tmp_path / "use.cpp"
    src.write_text(
        '#include "lmra_b200.hpp"\n'
        "int main() {\n"
        "  lmra::AlgoConfig cfg; cfg.rank = lmra::MultilinearRank({2, 2, 2});\n"
        "  auto c = lmra::amm_sample_counts({6, 6, 6}, cfg, true);\n"
        "  if (c.size() != 3) return 1;\n"
        "  lmra::DenseTensor t({2, 3}, {1, 2, 3, 4, 5, 6.5});\n"
        f"  lmra::save_tensor(\"{tmp_path}/t.tnsr\", t);\n"
        f"  lmra::DenseTensor u = lmra::load_tensor(\"{tmp_path}/t.tnsr\");\n"
        "  if (u.dims() != t.dims() || u.data()[5] != 6.5) return 2;\n"
        "  if (lmra::all_algorithm_ids().size() != 9 || lmra::algorithm_id(lmra::Algorithm::Hooi) != \"hooi\") return 5;\n"
        "  if (!lmra::parse_algorithm(\"alg5\") || lmra::parse_algorithm(\"alg3\")) return 6;\n"
        "  if (lmra::thread_cap() < 1) return 7;\n"
        "  if (cfg.rank.clamped_for({1, 5, 5}) != std::vector<std::size_t>({1, 2, 2})) return 8;\n"
        "  try { cfg.rank.clamped_for({1, 5}); return 9; } catch (const std::invalid_argument&) {}\n"
        "  try { lmra::load_tensor(\"/nonexistent.tnsr\"); return 3; }\n"
        "  catch (const std::runtime_error& e) { return std::string(e.what()).find(\"cannot open\") == 0 ? 0 : 4; }\n"
        "}\n")
    exe = tmp_path / "use"
    lib_dir = os.path.join(ROOT, "paper_2303_11612_b200", "lib")
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                    "-L", lib_dir, "-llmra_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    assert subprocess.run([str(exe)]).returncode == 0  # host-only call: works without a GPU
