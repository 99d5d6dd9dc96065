"""Runs single ls_expand cases (R n1 n2 n3 k0 k1 pad_y pad_z) and synchronizes after each, so a
failing case is named (lab triage of fuzz_long.py failures).

  python tools/lab/repro_case.py 32,93,236,4,3,4,5,0 [more cases ...]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import torch  # noqa: E402

from paper_1405_2270_b200 import _abi  # noqa: E402

lib = _abi.load()
dev = torch.device("cuda")
p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
for spec in sys.argv[1:]:
    R, n1, n2, n3, k0, k1, pad_y, pad_z = map(int, spec.split(","))
    fac = [torch.rand((R, m), dtype=torch.float64, device=dev) * 0.95 + 0.05 for m in (n1, n2, n3)]
    w = torch.rand(R, dtype=torch.float64, device=dev) * 0.95 + 0.05
    ldy, nk = n1 + pad_y, k1 - k0
    ldz = ldy * n2 + pad_z
    buf = torch.full((nk * ldz + 8,), float("nan"), dtype=torch.float64, device=dev)
    buf2 = torch.empty(64, dtype=torch.float64, device=dev)
    name = C.create_string_buffer(256)
    lib.ls_expand_plan_name(R, name, 256)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = lib.ls_expand(p(fac[0]), n1, p(fac[1]), n2, p(fac[2]), n3, p(w), n1, n2, n3, R, k0, k1, p(buf), ldy, ldz,
                       None, None, None, None, s)
    print(spec, "rc", rc, name.value.decode(), flush=True)
    torch.cuda.synchronize()
    got = buf[: nk * ldz].view(nk, ldz)[:, : ldy * n2].reshape(nk, n2, ldy)[:, :, :n1]
    want = torch.einsum("q,qi,qj,qk->kji", w, fac[0], fac[1], fac[2][:, k0:k1])
    print("   rel", float((got - want).abs().max() / want.abs().max()), flush=True)
