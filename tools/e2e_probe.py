import sys, time, ctypes as C, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, ".")
import bench
from paper_1606_07822_b200 import api
from paper_1606_07822_b200._lib import CgTrainStats, check, load, ptr
for name in sys.argv[1:]:
    c, vocab, ids = bench.workload(name, 0, 1)
    tree = api.build_huffman_tree(vocab); sel = api.select_cached_nodes(tree, 31)
    cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=1, cache_nodes=31, seed=c.seed, mode="hogwild")
    keep=[]; desc = api.model_desc(vocab, tree, sel, keep); ccfg = cfg.to_c()
    ids_pin = torch.from_numpy(ids).pin_memory()
    out0 = torch.empty((vocab.size(), c.dim)).pin_memory(); out1 = torch.empty((vocab.size()-1, c.dim)).pin_memory()
    for r in range(4):
        st = CgTrainStats(); t0=time.perf_counter()
        check(load().cg_train(C.byref(ccfg), 0, C.byref(desc), ptr(ids_pin.numpy(), C.c_int32), ids.size, ptr(out0.numpy(), C.c_float), ptr(out1.numpy(), C.c_float), C.byref(st)))
        print(name, r, f"wall {time.perf_counter()-t0:.4f}s kernel {st.kernel_seconds:.4f}s lib-wall {st.wall_seconds:.4f}", flush=True)
