"""cachegram-b200: skip-gram hierarchical-softmax training with hot-node caching
(arXiv 1606.07822) as hand-written sm_100a CUDA behind the reference's train() API.

The product is libcachegram_b200.so (C-ABI: include/cachegram_b200.h; C++ drop-in:
include/cachegram/*.hpp). This package is its Python binding (``api``), the
synthetic corpus generators used by the benchmark (``corpus_gen``) and the
multi-GPU replica driver (``replicas``).
"""
from .api import (  # noqa: F401
    CacheSelection,
    HuffmanTree,
    Model,
    NodeCache,
    Session,
    TrainConfig,
    TrainStats,
    Vocabulary,
    build_huffman_tree,
    build_vocabulary_file,
    init_model,
    keep_probability,
    read_id_stream,
    select_cached_nodes,
    sigmoid_table,
    train,
    train_center,
    update_alpha,
)
