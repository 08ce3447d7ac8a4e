import torch, time
n = 100_000_000
F = torch.zeros(n, dtype=torch.float64, device="cuda")
k = 23_000_000
t = torch.randint(0, n, (k,), device="cuda", dtype=torch.int64)
v = torch.rand(k, device="cuda", dtype=torch.float64)
def tm(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - a)
    return best * 1e3
print("unsorted index_add_ %.3f ms" % tm(lambda: F.index_add_(0, t, v)))
ts, order = torch.sort(t)
vs = v[order]
print("sorted   index_add_ %.3f ms" % tm(lambda: F.index_add_(0, ts, vs)))
print("sort itself (torch.sort 23M int64) %.3f ms" % tm(lambda: torch.sort(t)))
# bucketed by high bits (4096 buckets), random within bucket
b = t >> 15
bo = torch.argsort(b, stable=False)
tb, vb = t[bo], v[bo]
print("bucketed(4096) index_add_ %.3f ms" % tm(lambda: F.index_add_(0, tb, vb)))
b2 = t >> 19
bo2 = torch.argsort(b2)
tb2, vb2 = t[bo2], v[bo2]
print("bucketed(256)  index_add_ %.3f ms" % tm(lambda: F.index_add_(0, tb2, vb2)))
