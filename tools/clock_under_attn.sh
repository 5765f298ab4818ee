nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/clk_attn.csv &
P=$!
python - <<'PY'
import ctypes, torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2602_00482_b200 import _native
lib=_native.lib(); vp=ctypes.c_void_p
n,S,H,dh=32768,1024,14,64; d=H*dh; rows=S+n
lib.tt_debug_attn_set_segments(16)
q=torch.randn(n,d,device="cuda").bfloat16(); K=torch.randn(rows,d,device="cuda").bfloat16(); V=torch.randn(rows,d,device="cuda").bfloat16()
dO=torch.randn(n,d,device="cuda").bfloat16(); o=torch.empty(n,d,device="cuda",dtype=torch.bfloat16)
lse=torch.empty(H,n,device="cuda"); D=torch.empty(H,n,device="cuda"); dq=torch.empty(n,d,device="cuda"); dk=torch.zeros(rows,d,device="cuda"); dv=torch.zeros(rows,d,device="cuda")
p=lambda t: vp(t.data_ptr()); ms=ctypes.c_float()
import time
for name, dirn, args in (("fwd",0,(vp(0),)*5),("bwd",1,(p(dO),p(D),p(dq),p(dk),p(dv)))):
    t=time.time()
    lib.tt_debug_attn(1,dirn,p(q),p(K),p(V),p(o),p(lse),*args,n,S,H,dh,ctypes.c_long(rows),2000 if dirn==0 else 1000,ctypes.byref(ms))
    print(name, ms.value, "ms", time.time()-t, flush=True)
PY
kill $P
