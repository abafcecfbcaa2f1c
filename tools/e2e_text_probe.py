"""Phase timing of train(corpus_path) (cg_train_file) on a bench config written as text:
python tools/e2e_text_probe.py c2   (run with CG_PROFILE=1 for the library's phase lines)."""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
from paper_1606_07822_b200 import api  # noqa: E402

for name in sys.argv[1:]:
    c, vocab, ids = bench.workload(name, 0, 1)
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=1,
                          cache_nodes=31, seed=c.seed, mode="hogwild")
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "c.txt")
        bench.write_text(bench.host_ids(ids), [vocab.word(i) for i in range(vocab.size())], path, len(ids))
        for r in range(3):
            t0 = time.perf_counter()
            api.train(path, vocab, tree, sel, cfg)
            print(name, r, f"api.train wall {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
