import ctypes as C, sys, time
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import torch
import bench
from paper_1408_5526_b200 import _lib
lib=_lib.lib(); st=_lib.stream_ptr()
dim=360; npts=bench.WORKLOADS["c4"][4]
out=torch.empty(1,dtype=torch.float64,device="cuda")
for gen in ("rasrap-recursive","philox"):
  for it in range(5):
    torch.cuda.synchronize(); t0=time.perf_counter()
    h=C.c_void_p(); _lib.check(lib.rq_sampler_create(C.byref(h), _lib.GEN_IDS[gen], dim, bench.SEED, 0, 1, st))
    torch.cuda.synchronize(); t1=time.perf_counter()
    _lib.check(lib.rq_stream_normals(h, 0, npts, out.data_ptr(), None, st))
    t2=time.perf_counter()
    v=float(out.item()); t3=time.perf_counter()
    lib.rq_sampler_destroy(h); t4=time.perf_counter()
    print(gen, it, 'create %.2f launch %.2f wait %.2f destroy %.2f total %.2f ms'%((t1-t0)*1e3,(t2-t1)*1e3,(t3-t2)*1e3,(t4-t3)*1e3,(t4-t0)*1e3))
