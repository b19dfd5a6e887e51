"""CPU: the C-ABI library loads and exports exactly what include/*.h declares;
host-side validation and accounting logic behave like the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracles import ROOT

kb = pytest.importorskip("paper_2402_02750_b200")


def header_functions(path):
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(kivi_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_header_symbol():
    L = kb.lib()
    declared = header_functions(os.path.join(ROOT, "include", "kivi_b200.h"))
    assert declared, "no functions parsed from the header"
    assert declared == set(kb.HEADER_SYMBOLS), declared ^ set(kb.HEADER_SYMBOLS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.kivi_abi_version() == 1


def test_library_is_sm100a_cuda_code():
    """The product .so carries sm_100a SASS (no PTX-only / CPU build)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump absent")
    out = subprocess.run(["cuobjdump", "--list-elf", kb.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("cfg,err", [
    ((2, 32, 128, 128), None), ((2, 32, 100, 64), kb.ConfigError), ((2, 32, 128, 50), kb.ConfigError),
    ((3, 2, 4, 2), kb.ConfigError), ((0, 2, 4, 2), kb.ConfigError), ((9, 2, 4, 2), kb.ConfigError),
    ((2, 0, 4, 2), kb.ConfigError), ((2, 2, 0, 2), kb.ConfigError), ((8, 4, 8, 4), None),
])
def test_config_validation_matches_reference(cfg, err):
    # reference CacheConfig::validate (kv_cache.cpp:7-21) + packable (quantize.cpp:173-176)
    c = kb.CacheConfig(*cfg)
    if err is None:
        c.validate()
    else:
        with pytest.raises(err):
            c.validate()
        assert kb.lib().kivi_last_error()


def test_error_message_is_thread_local_and_specific():
    with pytest.raises(kb.ConfigError, match="residual_length 100 must be divisible"):
        kb.CacheConfig(2, 32, 100, 64).validate()


def test_bench_bytes_formula_matches_survey():
    """SURVEY §8d per-unit bytes at config 1 (l=4096): 582,656 B."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert bench.attend_bytes_per_unit(4096, 2) == 582656
    # C3 (ctx 8192, 4 q-heads per kv-head): 1,110,016 B
    assert bench.attend_bytes_per_unit(8192, 2, qpk=4) == 1110016
    # C5 (ctx 32768): 4,252,672 B
    assert bench.attend_bytes_per_unit(32768, 2) == 4252672


def test_memory_accounting_closed_form():
    """reference memory_bytes (kv_cache.cpp:110-127): packed bytes + 4 B per
    group + 2 B per residual element at the high-water capacity.  The C port
    reproduces the reference's counters (goldens); here the closed form the
    library uses (kivi_cache_get_info) is checked against the port."""
    from oracles import Port
    p = Port()
    rng = np.random.default_rng(5)
    for bits, G, R, d, l in ((2, 32, 128, 128, 4000), (4, 4, 8, 8, 19), (2, 2, 2, 2, 1)):
        u = p.unit(bits, G, R, d)
        u.prefill(rng.uniform(-1, 1, (l, d)), rng.uniform(-1, 1, (l, d)))
        for _ in range(R + 1):
            u.append(rng.uniform(-1, 1, d), rng.uniform(-1, 1, d))
        c = u.counters()
        L = l + R + 1
        kg, vg = L - L % R, L - min(L, R)
        assert (c["key_grouped"], c["value_grouped"]) == (kg, vg)

        def grouped(tok):
            return (tok * d * bits + 7) // 8 + 4 * (tok * d // G)
        assert c["key_memory"] == grouped(kg) + 2 * c["key_capacity"] * d
        assert c["value_memory"] == grouped(vg) + 2 * c["value_capacity"] * d
        assert c["key_capacity"] == R and c["value_capacity"] == R


def test_no_gpu_create_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    c = kb.CacheConfig(2, 32, 128, 128)._c()
    rc = kb.lib().kivi_cache_create(ctypes.byref(c), 0, 4, 256, ctypes.byref(h))
    assert rc in (4, 5)  # CUDA error / OOM, never a crash or a silent CPU path
    assert not h.value


def test_facade_library_exports_reference_api():
    """The C++ drop-in facade exports the reference's kivi:: entry points."""
    import shutil
    import subprocess
    path = kb.FACADE_PATH
    if not os.path.exists(path):
        pytest.skip("facade not built")
    if not shutil.which("nm"):
        pytest.skip("nm absent")
    syms = subprocess.run(["nm", "-DC", path], capture_output=True, text=True).stdout
    for sym in ("kivi::prefill(", "kivi::append_token(", "kivi::decode_attention(",
                "kivi::reference_attention(", "kivi::materialize_keys(",
                "kivi::materialize_values(", "kivi::memory_bytes(", "kivi::quantize_group(",
                "kivi::dequantize_group(", "kivi::pack_codes(", "kivi::unpack_codes(",
                "kivi::QuantizedTensor::quantize(", "kivi::QuantizedTensor::dequantize(",
                "kivi::QuantizedTensor::concat_tokens(", "kivi::CacheConfig::validate("):
        assert sym in syms, sym


def test_driver_library_exports_its_header():
    """libkivi_driver.so (the C++ decode driver) exports include/kivi_driver.h."""
    from paper_2402_02750_b200 import workload as wl
    declared = header_functions(os.path.join(ROOT, "include", "kivi_driver.h"))
    assert declared == set(wl.DRIVER_SYMBOLS), declared
    L = wl.driver_lib()
    for name in declared:
        assert hasattr(L, name), name


def test_driver_validates_before_touching_a_device():
    """Spec/config errors come back as the reference's exception types with no GPU."""
    from paper_2402_02750_b200 import workload as wl
    sp = wl.WorkloadSpec(batch=1, prompt_len=4, gen_len=1, layers=1, kv_heads=1, head_dim=64)
    with pytest.raises(kb.ConfigError):   # fused projection needs head_dim 128
        wl.run_decode_benchmark_native(sp, kb.CacheConfig(2, 32, 128, 64))
    with pytest.raises(kb.ConfigError):   # workload counts must be >= 1
        wl.run_decode_benchmark_native(wl.WorkloadSpec(batch=0, head_dim=128),
                                       kb.CacheConfig(2, 32, 128, 128))
