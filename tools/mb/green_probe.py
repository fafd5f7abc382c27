"""Green-context probe (CUDA 12.x driver API via cuda-python): can a stream
of a green context with a subset of the SMs run kernels on memory allocated
by the primary context (torch / our library), and are its kernels confined to
those SMs?  Prints one JSON line."""

import json
import time

import torch
import cuda.bindings.driver as d


def ok(r):
    err = r[0] if isinstance(r, tuple) else r
    assert err == d.CUresult.CUDA_SUCCESS, r
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) and len(r) == 2 else None)


torch.cuda.init()
x = torch.randn(1 << 26, device="cuda")
ok(d.cuInit(0))
dev = ok(d.cuDeviceGet(0))
res = ok(d.cuDeviceGetDevResource(dev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
total = res.sm.smCount
out = {"sm_total": total}
for want in (16, 32):
    groups, n, rem = ok(d.cuDevSmResourceSplitByCount(1, res, 0, want))
    desc = ok(d.cuDevResourceGenerateDesc([groups[0]], 1))
    g = ok(d.cuGreenCtxCreate(desc, dev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    s = ok(d.cuGreenCtxStreamCreate(g, d.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    ext = torch.cuda.ExternalStream(int(s))
    torch.cuda.synchronize()
    with torch.cuda.stream(ext):
        y = x * 2.0 + 1.0  # warm
    ext.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(ext):
        for _ in range(20):
            y = torch.sin(x) * torch.cos(x)
    ext.synchronize()
    dt_g = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(20):
        z = torch.sin(x) * torch.cos(x)
    torch.cuda.synchronize()
    dt_p = time.perf_counter() - t0
    out[f"green_{want}"] = {"sm_count": groups[0].sm.smCount, "remaining": rem.sm.smCount,
                            "result_ok": bool(torch.equal(y, z)), "green_ms": dt_g * 1e3, "primary_ms": dt_p * 1e3}
print(json.dumps(out))
