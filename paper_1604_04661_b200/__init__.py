"""B200-native pSGNScc (arXiv 1604.04661): minibatched skip-gram negative sampling
with shared negatives, as a drop-in for the reference `sgns` package's training
entry points, per-minibatch operator and data-parallel loop.

The hot path is CUDA C++ for sm_100a behind a C ABI (include/sgns_b200.h,
libsgns_b200.so in this directory); there is no CPU fallback.
"""

from .corpus import (EncodedCorpus, NegativeTable, Vocabulary, build_negative_table, build_vocab,
                     build_vocab_file, encode_corpus, encode_corpus_file, keep_probability,
                     partition_sentences, read_tokens, split_by_tokens)
from .distributed import (DistributedRunError, HostStagedTransport, NcclTransport, SyncPolicy, Transport,
                          TransportError, distributed_train, partition_corpus, scaled_alpha0,
                          select_sync_rows)
from .kernel_batched import Minibatch, WindowBatch, process_batch, update_windows
from .model import (DeviceModel, EmbeddingModel, ModelFormatError, detect_format, init_device_model,
                    init_model, load_debug, load_model, save_debug, save_model, sigmoid)
from .trainer import (ConfigError, DeviceRun, TrainingConfig, TrainingStats, train,
                      train_encoded, update_alpha)

__version__ = "0.1.0"

__all__ = [
    "ConfigError", "DeviceModel", "DeviceRun", "DistributedRunError", "EmbeddingModel",
    "EncodedCorpus", "HostStagedTransport", "Minibatch", "NcclTransport", "NegativeTable", "SyncPolicy",
    "TrainingConfig", "TrainingStats", "Transport", "TransportError", "Vocabulary",
    "WindowBatch", "build_negative_table", "build_vocab", "distributed_train", "encode_corpus",
    "init_device_model", "init_model", "keep_probability", "partition_corpus", "save_model",
    "load_model", "detect_format", "save_debug", "load_debug", "ModelFormatError",
    "build_vocab_file", "encode_corpus_file",
    "partition_sentences", "process_batch", "read_tokens", "scaled_alpha0", "select_sync_rows",
    "sigmoid", "split_by_tokens", "train", "train_encoded", "update_alpha", "update_windows",
]
