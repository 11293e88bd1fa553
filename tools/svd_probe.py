import torch, time, json
res = {}
for l in (144, 272, 420):
    g = torch.Generator(device="cuda").manual_seed(0)
    R = torch.triu(torch.randn(l, l, generator=g, dtype=torch.float64, device="cuda"))
    for name, fn in [("gesvd", lambda: torch.linalg.svd(R, driver="gesvd")),
                     ("gesvdj", lambda: torch.linalg.svd(R, driver="gesvdj")),
                     ("gesvda", lambda: torch.linalg.svd(R, driver="gesvda")),
                     ("eigh", lambda: torch.linalg.eigh(R.T @ R))]:
        try:
            for _ in range(2): fn()
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(5): fn()
            torch.cuda.synchronize()
            res[f"{name}_{l}_ms"] = (time.perf_counter() - t) / 5 * 1e3
        except Exception as e:
            res[f"{name}_{l}_ms"] = str(e)[:80]
print(json.dumps(res, indent=1))
