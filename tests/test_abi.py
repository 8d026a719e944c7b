"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/rl_policy.h
declares, and rejects host-detectable bad arguments before enqueueing anything (so these
calls never reach the device)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2605_15565_b200 as rl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rl_policy.h")


def _header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rl_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(rl.lib_path()):
        from paper_2605_15565_b200 import build
        build.build()
    return rl.load()


def test_library_exports_every_header_symbol(lib):
    declared = _header_functions()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", rl.lib_path()], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (rl_[a-z0-9_]+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    assert set(declared) == set(rl.EXPORTED_SYMBOLS)


def test_sm100a_cubin_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", rl.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in ln for ln in out.splitlines() if ".cubin" in ln)


def test_status_strings_and_version(lib):
    assert lib.rl_abi_version() == 2
    assert lib.rl_status_string(0) == b"ok"
    assert lib.rl_status_string(1) == b"invalid-argument"
    assert lib.rl_status_string(6) == b"nccl-error"


def test_params_default(lib):
    p = rl._Params()
    lib.rl_loss_params_default(C.byref(p))
    assert abs(p.clip_eps_low - 0.2) < 1e-7 and abs(p.clip_eps_high - 0.2) < 1e-7
    assert p.inv_temperature == 1.0 and p.log_ratio_clamp == 20.0 and p.max_staleness == -1
    assert p.agg == rl.AGG_TOKEN_MEAN and p.active_tokens_dev is None
    assert p.kl_coef == 0.0 and p.ref_logp is None and p.prox_logp is None
    # the ctypes mirror matches the C layout (size and every field offset), compiled from the header
    import shutil
    import subprocess
    import tempfile
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    fields = [f for f, _ in rl._Params._fields_]
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"rl_policy.h\"\nint main(void){printf(\"%zu\", sizeof(rl_loss_params));"
    src += "".join(f'printf(" %zu", offsetof(rl_loss_params, {f}));' for f in fields) + "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        with open(os.path.join(d, "t.c"), "w") as fh:
            fh.write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", os.path.join(d, "t"),
                        os.path.join(d, "t.c")], check=True)
        vals = [int(v) for v in subprocess.run([os.path.join(d, "t")], capture_output=True, text=True,
                                               check=True).stdout.split()]
    assert vals[0] == C.sizeof(rl._Params)
    assert vals[1:] == [getattr(rl._Params, f).offset for f in fields]


def test_host_validation_rejects_before_launch(lib):
    fake = 0x10000  # never dereferenced: validation fails first
    # ld < vocab
    assert lib.rl_token_logprob(fake, rl.BF16, 4, 100, 96, fake, 1.0, fake, None, None, None) == 1
    # misaligned logits
    assert lib.rl_token_logprob(fake + 2, rl.BF16, 4, 96, 96, fake, 1.0, fake, None, None, None) == 2
    # ld * 2 bytes not a multiple of 16
    assert lib.rl_token_logprob(fake, rl.BF16, 4, 90, 92, fake, 1.0, fake, None, None, None) == 2
    # bad dtype / temperature
    assert lib.rl_token_logprob(fake, 7, 4, 96, 96, fake, 1.0, fake, None, None, None) == 1
    assert lib.rl_token_logprob(fake, rl.BF16, 4, 96, 96, fake, 0.0, fake, None, None, None) == 1
    assert b"inv_temperature" in lib.rl_last_error()
    p = rl.LossParams()._c()
    # workspace too small
    assert lib.rl_policy_loss_fwd_bwd(fake, rl.BF16, 4, 96, 96, fake, fake, None, fake, fake, None,
                                      None, C.byref(p), fake, None, None, fake, fake, 8, None) == 4
    # kl_coef without ref_logp
    p.kl_coef = 1e-3
    assert lib.rl_policy_loss_fwd_bwd(fake, rl.BF16, 4, 96, 96, fake, fake, None, fake, fake, None,
                                      None, C.byref(p), fake, None, None, fake, fake, 1 << 20, None) == 1
    assert b"ref_logp" in lib.rl_last_error()
    p.kl_coef = 0.0
    # SEQ_MEAN without seq_active
    p.agg = rl.AGG_SEQ_MEAN_TOKEN_MEAN
    ws = lib.rl_policy_loss_workspace_size(4, 96, rl.BF16)
    assert lib.rl_policy_loss_fwd_bwd(fake, rl.BF16, 4, 96, 96, fake, fake, None, fake, fake, None,
                                      None, C.byref(p), fake, None, None, fake, fake, ws, None) == 1
    # partial overlap of dlogits with logits
    p.agg = rl.AGG_TOKEN_MEAN
    assert lib.rl_policy_loss_fwd_bwd(fake, rl.BF16, 4, 96, 96, fake, fake, None, fake, fake, None,
                                      None, C.byref(p), fake + 64, None, None, fake, fake, ws,
                                      None) == 1
    # advantages: bad std mode, batch norm without workspace
    assert lib.rl_group_advantage(fake, fake, 1, 8, 9, 1e-6, 0, 1e-6, None, None, 0, fake, None, None) == 1
    assert lib.rl_group_advantage(fake, fake, 1, 8, 0, 1e-6, 1, 1e-6, fake, None, 0, fake, None, None) == 4
    # bookkeeping: tokens without sequences
    assert lib.rl_seq_bookkeeping(fake, 0, 5, None, fake, 10, None, 0, -1, None, fake, fake, None,
                                  None, None, None, None) == 1
    # vocab-parallel without comm
    assert lib.rl_vocab_parallel_logprob(fake, rl.BF16, 4, 96, 0, 96, 96, fake, 1.0, None, fake,
                                         None, None, None, None, None, None, None, None, None, None,
                                         fake, 1 << 20, None) == 1


def test_refuses_to_enqueue_without_an_sm100_device(lib):
    """A call that passes every host check reaches the device check, which answers
    RL_ERR_UNSUPPORTED on anything but a compute-capability 10.0 device (here: no device)."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present: the fake pointers below would be dereferenced")
    fake = 0x10000
    assert lib.rl_token_logprob(fake, rl.BF16, 4, 96, 96, fake, 1.0, fake, None, None, None) == 3
    assert b"sm_100a" in lib.rl_last_error()


def test_zero_sized_calls_are_noops(lib):
    assert lib.rl_group_advantage(None, None, 0, 0, 0, 1e-6, 0, 1e-6, None, None, 0, None, None, None) == 0
    assert lib.rl_token_logprob(None, rl.BF16, 0, 8, 8, None, 1.0, None, None, None, None) == 0


def test_binding_refuses_cpu_tensors(lib):
    torch = pytest.importorskip("torch")
    x = torch.zeros(4, 8)
    with pytest.raises(rl.RLError):
        rl.token_logprob(x, torch.zeros(4, dtype=torch.int32), torch.zeros(4))


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2605_15565_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f


def test_dev_options_header_matches_binding(lib):
    """include/rl_policy_dev.h and the binding's DEV_* constants name the same option keys, and the
    library accepts exactly those keys (an unknown key answers -1 and changes nothing)."""
    src = open(os.path.join(ROOT, "include", "rl_policy_dev.h")).read()
    keys = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define RL_DEV_([A-Z0-9_]+) (\d+)", src)}
    assert keys, "no RL_DEV_* keys in the header"
    for name, k in keys.items():
        assert getattr(rl, "DEV_" + name) == k, name
        old = lib.rl_dev_set_option(k, 0)
        assert old >= 0 and lib.rl_dev_set_option(k, old) == 0
    assert lib.rl_dev_set_option(max(keys.values()) + 1, 1) == -1
