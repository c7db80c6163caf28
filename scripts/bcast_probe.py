"""Fused output broadcast (bps_apply_orbit_range_bcast) on one GPU: cost of the epilogue stores to
extra destinations (stand-ins for the peers' symmetric buffers) vs the plain orbit-range apply, and
whether torch symmetric memory exposes an NVLS multicast address on this platform."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2602_06071_b200 import Sketch, configs as C, dist as D

os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cfg = C.GRAD.with_(n=int(os.environ.get("BN_COLS", "1024")))
sk = Sketch(**cfg.sketch_args())
A = torch.randn((cfg.d, cfg.n), device="cuda", dtype=torch.bfloat16)
M, B_r = sk.M, sk.B_r
A_loc = torch.cat([A, A[:(sk.kappa - 1) * sk.B_c]])  # orbit-local stand-in of the right size (timing only)
Yl = torch.empty((M * B_r, cfg.n), device="cuda")
buf, ptrs, mc, barrier = D.symmetric_rendezvous((M * B_r, cfg.n), A.device)
res = {"config": f"grad sketch, n={cfg.n}", "symmetric_ptrs": len(ptrs), "multicast_ptr": bool(mc)}
dsts = [torch.empty((M * B_r, cfg.n), device="cuda") for _ in range(7)]

def t(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it

res["plain_ms"] = t(lambda: sk.apply_orbit_range(0, M, A_loc, out=Yl))
res["bcast_symm_ms"] = t(lambda: sk.apply_orbit_range(0, M, A_loc, out=Yl, dst=ptrs, dst_ld=cfg.n))
res["bcast_1_local_ms"] = t(lambda: sk.apply_orbit_range(0, M, A_loc, out=Yl, dst=[dsts[0].data_ptr()], dst_ld=cfg.n))
res["bcast_7_local_ms"] = t(lambda: sk.apply_orbit_range(0, M, A_loc, out=Yl, dst=[d.data_ptr() for d in dsts], dst_ld=cfg.n))
if mc:
    res["bcast_multicast_ms"] = t(lambda: sk.apply_orbit_range(0, M, A_loc, out=Yl, mc_ptr=mc, dst_ld=cfg.n))
    torch.cuda.synchronize(); barrier(); torch.cuda.synchronize()
    res["multicast_bitwise"] = bool(torch.equal(buf, Yl))
import ctypes
from paper_2602_06071_b200._lib import lib
def split(fn):
    lib.bps_timing_enable(1)
    for _ in range(5): fn()
    torch.cuda.synchronize(); lib.bps_timing_enable(0)
    tot, cnt = ctypes.c_double(), ctypes.c_uint64()
    lib.bps_timing_read(ctypes.byref(tot), ctypes.byref(cnt)); main = tot.value / max(1, cnt.value)
    lib.bps_timing_read_ex(1, ctypes.byref(tot), ctypes.byref(cnt)); aux = tot.value / 5
    return round(main, 4), round(aux, 4)
res["plain_main_aux_ms"] = split(lambda: sk.apply_orbit_range(0, M, A_loc, out=Yl))
res["bcast1_main_aux_ms"] = split(lambda: sk.apply_orbit_range(0, M, A_loc, out=Yl, dst=[dsts[0].data_ptr()], dst_ld=cfg.n))
res["sparse_bcast_1_ms"] = t(lambda: sk.apply_orbit_range(0, M, A_loc[:, :64].contiguous(), out=Yl[:, :64], dst=[dsts[0].data_ptr()], dst_ld=cfg.n, variant="sparse"), 2)
print(json.dumps(res))
dist.destroy_process_group()
