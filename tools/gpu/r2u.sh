for lib in libfhv_exp.so libfhv_b200.so; do
python - <<PY
import os, torch, time
os.environ["FHV_LIB"]="$PWD/paper_2211_15460_b200/$lib"
import paper_2211_15460_b200 as fhv
from paper_2211_15460_b200 import _lib
import bench
w=bench.workload()
s=w["scene"]; dev=torch.device("cuda",0)
counts=torch.randint(0,40,(8**8,),dtype=torch.int32,device=dev).view(torch.uint32)
offs=torch.empty_like(counts); pyr=torch.empty(((8**8-1)//7,),dtype=torch.uint8,device=dev)
lib=_lib.load(); c=_lib.ctx(dev)
import ctypes
fn=lib.fhv_pofa_shard_directory
fn.argtypes=[ctypes.c_void_p,ctypes.c_int32,ctypes.c_void_p,ctypes.c_void_p,ctypes.c_void_p,ctypes.c_void_p,ctypes.c_uint64,ctypes.c_void_p]
# fhv_pofa_shard_directory needs pass1 state; use the internal scan via a POFA build instead: time via prof
def b():
    try: fhv.pofa_build(s,w["strategy"],w["cfg"],8,device=dev)
    except Exception: pass
b()
_lib.prof_enable(dev,True); _lib.prof_collect(dev)
for _ in range(20): b()
torch.cuda.synchronize()
p=_lib.prof_collect(dev)
print("$lib", {k:round(v[0]/v[1],4) for k,v in p.items() if k in ("scan_leaves",)})
PY
done
