import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch
import paper_2402_12274_b200 as mp
inst = mp.init(group="p1", device=0)
q = mp.queue_create(inst)
info = mp.info_create(); info.set("type", "devstream"); mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
s = inst.stream_create(info); c = mp.stream_comm_create(inst.world, s)
count = 16 << 20
x = torch.full((count,), 1.0, device=inst.device); y = torch.zeros_like(x)
for _ in range(3):
    mp.allreduce_enqueue(c, x, y, count, mp.FLOAT32, algo="native")
mp.queue_synchronize(q)
print("ok", float(y[0]))
mp.comm_free(c); mp.free_stream(s); inst.finalize()
