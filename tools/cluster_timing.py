import time, json, sys
sys.path.insert(0, '.')
import torch, numpy as np
import paper_2507_21253_b200 as B
out = {}
for cfg in (2, 5):
    a = B.make_config(cfg)
    e = B.Engine(0)
    A = e.upload(a); At = e.transpose(A)
    for rep in range(2):
        t0 = time.perf_counter(); p = e.spgemm_topk(A, At, 7, 0.3); e.synchronize(); t_tk = time.perf_counter() - t0
        t0 = time.perf_counter(); q = e.minhash_candidates(A, 64, 32, 1, 7, 0.3); e.synchronize(); t_mh = time.perf_counter() - t0
    t0 = time.perf_counter(); asg = B.merge_candidates(a, p); t_merge = time.perf_counter() - t0
    t0 = time.perf_counter(); asg2 = e.hierarchical_clusters(a, method="minhash", nhash=64); t_full_mh = time.perf_counter() - t0
    t0 = time.perf_counter(); asg3 = e.hierarchical_clusters(a); t_full_tk = time.perf_counter() - t0
    out[f"cfg{cfg}"] = dict(topk_candidates_s=t_tk, minhash_candidates_s=t_mh, npairs_topk=int(p.size), npairs_minhash=int(q.size),
                          host_merge_s=t_merge, hierarchical_topk_s=t_full_tk, hierarchical_minhash_s=t_full_mh,
                          clusters_topk=asg3.nclusters, clusters_minhash=asg2.nclusters)
    e.close()
print(json.dumps(out))
