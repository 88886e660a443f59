import torch, json
dev = torch.device("cuda", 0)
x = torch.empty(4243648 * 32, dtype=torch.float32, device=dev).view(-1, 32)   # 543 MB of 128-B lines
n = x.shape[0]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
def t(fn, reps=5):
    fn(); ts = []
    for _ in range(reps):
        flush.zero_(); torch.cuda._sleep(100000)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts)//2]
for m in (262144, 1048576):
    idx = torch.randint(0, n, (m,), device=dev)
    ms = t(lambda: x.index_select(0, idx))
    res["random_lines_%d" % m] = {"ms": ms, "GBs_read": m * 128 / ms / 1e6}
    # strided: every 16th line (2 KB stride) like x-faces
    idx2 = (torch.arange(m, device=dev) * 16) % n
    ms = t(lambda: x.index_select(0, idx2))
    res["stride2KB_lines_%d" % m] = {"ms": ms, "GBs_read": m * 128 / ms / 1e6}
y = torch.empty(256 << 20, dtype=torch.uint8, device=dev); z = torch.empty_like(y)
ms = t(lambda: z.copy_(y)); res["copy256MB"] = {"ms": ms, "GBs_rw": 2 * y.numel() / ms / 1e6}
print(json.dumps(res))
