import sys, numpy as np
sys.path.insert(0, '.')
from paper_2102_05221_b200 import ingest, series
rng = np.random.default_rng(1)
for name, xs in [("small", [np.arange(5.0), np.arange(7.0)]), ("const", [np.full(10, 3.25)]), ("long", [rng.normal(size=200000).cumsum()]), ("mid", [rng.normal(size=3000) for _ in range(5)])]:
    for op in ("derivative", "znormalize"):
        try:
            with ingest.DeviceSeries.upload(xs) as d:
                with getattr(d, op)() as o:
                    got = o.to_host()
            want = [getattr(series, op)(x) for x in xs]
            print(name, op, all(a.tobytes() == b.tobytes() for a, b in zip(got, want)), flush=True)
        except Exception as e:
            print(name, op, "ERR", e, flush=True)
            sys.exit(1)
