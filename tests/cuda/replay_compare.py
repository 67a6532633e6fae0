"""Long drop-in replays vs the pure reference simulator (manual validation;
the GPU test suite runs the 32-request case): every request's FTR / hits and
the eviction total must be identical."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from oracle.oracle import REF_DIR
from paper_2601_12967_b200 import dropin as D

ref_lib = os.path.join(REF_DIR, "libagentsim_ref.so")
for n, pool in ((256, 8192), (256, 2048), (512, 8192)):
    for preset in ("sutradhara", "baseline", "sutradhara_no_tiering"):
        kw = {"kv_tiering": 0} if preset.endswith("no_tiering") else {}
        p = "sutradhara" if preset.startswith("sutradhara") else preset
        try:
            ref = D.run_shard(n, 1, p, pool, shard=0, n_shards=1, lib_path=ref_lib, **kw)
            got = D.run_shard(n, 1, p, pool, shard=0, n_shards=1, **kw)
        except TypeError as e:
            print("skip", preset, e)
            continue
        same = (np.array_equal(ref.ftr_ms, got.ftr_ms) and np.array_equal(ref.hit_tokens, got.hit_tokens)
                and ref.evictions == got.evictions)
        print(n, pool, preset, "IDENTICAL" if same else "DIFFERENT", ref.evictions, got.evictions,
              round(ref.wall_s, 1), round(got.wall_s, 1), flush=True)
