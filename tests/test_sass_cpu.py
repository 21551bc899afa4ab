"""Static checks of the shipped sm_100a machine code (no GPU: cuobjdump on the built library).

They guard properties the parity tests can only catch by chance:
- every TMA-staged quantizer orders its shared-memory loads before the mbarrier arrive that lets
  TMA refill the buffer (a proxy fence in front of the release, round-2b race);
- the hot kernels are real tcgen05 / TMA code."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


@pytest.fixture(scope="module")
def sass():
    if not os.path.exists(CUOBJDUMP):
        pytest.skip("cuobjdump not available")
    from paper_2603_18742_b200 import build
    lib = build.build()
    out = subprocess.run([CUOBJDUMP, "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        if cur:
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
            if m:
                funcs[cur].append(m.group(1).strip())
    return funcs


def _kernels(sass, pat):
    ks = {k: v for k, v in sass.items() if re.search(pat, k)}
    assert ks, f"no kernel matches {pat}"
    return ks


def test_quantizer_release_after_proxy_fence(sass):
    """In every quant_had / quant_tma instantiation, the buffer-release arrive (plain, non-tx
    mbarrier arrive) comes after a FENCE.VIEW.ASYNC.S that follows the last shared-memory load
    before it: no LDS can still be in flight when TMA may overwrite the buffer."""
    n = 0
    for name, ins in _kernels(sass, r"quant_(had|tma)_kernel").items():
        arrives = [i for i, s in enumerate(ins) if re.search(r"SYNCS\.ARRIVE\.TRANS64\.A1T0", s)]
        assert arrives, f"{name}: no buffer-release arrive found"
        for a in arrives:
            lds = [i for i in range(a) if ins[i].split()[0].startswith("LDS") or " LDS" in ins[i]]
            fences = [i for i in range(a) if "FENCE.VIEW.ASYNC.S" in ins[i]]
            last_lds = max(lds) if lds else -1
            assert any(f > last_lds for f in fences), f"{name}: release arrive at {a} not fenced after LDS at {last_lds}"
            n += 1
    assert n >= 10


def test_gemm_kernels_are_tcgen05_tma(sass):
    """The GEMM instantiations issue 2-CTA tcgen05 MMAs (UTC*MMA.2CTA), read TMEM (LDTM) and move
    operands by TMA (UTMALDG); the NVFP4 one copies scale factors to TMEM (UTCCP)."""
    for name, ins in _kernels(sass, r"dmpq_gemm_pair_kernel").items():
        txt = "\n".join(ins)
        assert re.search(r"UTC\w*MMA\S*\.2CTA", txt), name
        assert "LDTM" in txt and "UTMALDG" in txt, name
        if re.search(r"pair_kernelILi1E", name):
            assert "UTCCP" in txt, name
