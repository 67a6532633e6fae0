import sys, time, os
sys.path.insert(0, "/root/repo")
from paper_2601_12967_b200 import dropin as D
from oracle.oracle import REF_DIR
n = int(os.environ.get("NREQ", "128"))
for preset in ("sutradhara",):
    t = time.time()
    kw = {"lib_path": os.path.join(REF_DIR, "libagentsim_ref.so")} if os.environ.get("REF") else {}
    r = D.run_shard(n, 1, preset, 8192, shard=0, n_shards=1, **kw)
    print(preset, "ref" if kw else "b200", "wall", round(time.time() - t, 2), "evictions", r.evictions,
          "ftr_sum", float(r.ftr_ms.sum()), "hit", float(r.hit_tokens.sum()), flush=True)
