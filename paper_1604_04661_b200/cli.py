"""`python -m paper_1604_04661_b200 train | train-dist | eval`.

Same flags and key:value reports as the reference CLI (sgns/cli.py:25-306), with the
GPU path underneath:
  * train: native ingestion -> device training -> word2vec file (byte-identical writer);
  * train-dist: one process per GPU over NCCL.  Under torchrun the rendezvous comes
    from the environment; the reference's socket-mode flags (-nodes/-rank/-hosts,
    "host:port" on the hosts file's first line) map to a TCP rendezvous instead.
    The reference's -inprocess N (threads sharing one process) has no GPU analogue:
    launch N processes with torchrun;
  * eval: similarity (device cosines) and analogy (device argmax GEMM).
New flags: -rng {philox,splitmix}, -workers N (device workers; default: all resident).
SGNS_FLOAT64=1 selects the float64 build as in the reference.  Exit codes: 0 ok,
1 runtime/data error (OSError, ValueError), 2 usage error.
"""

from __future__ import annotations

import argparse
import os
import socket
import sys


def write_report(path: str, items: dict) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for k, v in items.items():
            fh.write(f"{k}: {v}\n")


def _stats_items(stats) -> dict:
    out = {"words_processed": stats.words_processed, "words_read": stats.words_read,
           "wall_seconds": f"{stats.wall_seconds:.3f}",
           "throughput_words_per_sec": f"{stats.throughput_words_per_sec:.1f}",
           "final_alpha": f"{stats.final_alpha:.8f}"}
    out.update({f"loss_epoch_{i}": f"{x:.6f}" for i, x in enumerate(stats.loss_by_epoch, 1)})
    return out


def _env_items() -> dict:
    items = {"host": socket.gethostname(), "cpu_count": os.cpu_count()}
    try:
        import torch
        if torch.cuda.is_available():
            items["device"] = torch.cuda.get_device_name(torch.cuda.current_device())
    except Exception:  # noqa: BLE001 - the report must not fail on a probe
        pass
    return items


def _config(args):
    from .trainer import TrainingConfig
    return TrainingConfig(dim=args.size, window=args.window, negatives=args.negative,
                          subsample=args.sample, min_count=args.min_count, alpha0=args.alpha,
                          epochs=args.iter, threads=args.threads, batch_cap=args.batch_size,
                          kernel=args.kernel, seed=args.seed, rng=args.rng, workers=args.workers,
                          float64=os.environ.get("SGNS_FLOAT64") == "1")


def _config_items(cfg, corpus: str) -> dict:
    return {"corpus": corpus, "dim": cfg.dim, "window": cfg.window, "negatives": cfg.negatives,
            "sample": cfg.subsample, "min_count": cfg.min_count, "alpha0": cfg.alpha0,
            "epochs": cfg.epochs, "threads": cfg.threads, "batch_size": cfg.batch_cap,
            "kernel": cfg.kernel, "seed": cfg.seed, "float64": int(cfg.float64),
            "rng": cfg.rng, "workers": cfg.workers if cfg.workers is not None else "auto"}


def cmd_train(args) -> int:
    from .model import save_model
    from .trainer import train
    cfg = _config(args)
    model, vocab, stats = train(args.train, cfg)
    save_model(model, vocab, args.output, binary=bool(args.binary))
    if args.save_vocab:
        vocab.save(args.save_vocab)
    if args.report:
        write_report(args.report, {"command": "train", **_config_items(cfg, args.train),
                                   "vocab_size": vocab.size, "total_tokens": vocab.total_tokens,
                                   **_stats_items(stats), **_env_items()})
    print(f"saved {vocab.size} x {cfg.dim} vectors to {args.output}")
    return 0


def _init_process_group(args) -> None:
    import torch
    import torch.distributed as dist
    if "RANK" in os.environ and "WORLD_SIZE" in os.environ:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return
    if args.nodes is None or args.rank is None or args.hosts is None:
        raise SystemExit("train-dist needs torchrun (RANK/WORLD_SIZE) or -nodes/-rank/-hosts")
    with open(args.hosts, encoding="utf-8") as fh:
        host, _, port = fh.readline().split()[0].partition(":")
    local = args.rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", init_method=f"tcp://{host}:{port}", rank=args.rank,
                            world_size=args.nodes, device_id=torch.device("cuda", local))


def cmd_train_dist(args) -> int:
    import torch.distributed as dist
    from .corpus import build_vocab_file, encode_corpus_file
    from .distributed import DistributedRunError, NcclTransport, SyncPolicy, distributed_train
    from .model import save_model
    if args.inprocess is not None:
        print("-inprocess has no GPU analogue: launch one process per GPU with "
              "`python -m torch.distributed.run --nproc-per-node N -m paper_1604_04661_b200 "
              "train-dist ...`", file=sys.stderr)
        return 2
    cfg = _config(args)
    policy = SyncPolicy(period_words=args.sync_period, hot_rows=args.hot_rows,
                        rotation_chunk=args.rotation)
    _init_process_group(args)
    transport = NcclTransport()
    try:
        vocab = build_vocab_file(args.train, cfg.min_count)
        encoded = encode_corpus_file(args.train, vocab)
        try:
            model, stats = distributed_train(None, cfg, policy, transport, prebuilt=(vocab, encoded))
        except DistributedRunError as exc:
            print(f"distributed run failed: {exc}", file=sys.stderr)
            if args.report:
                write_report(args.report, {"command": "train-dist", "status": "aborted",
                                           "rank": transport.rank, **_stats_items(exc.partial_stats)})
            return 1
        if transport.rank == 0:
            save_model(model, vocab, args.output, binary=bool(args.binary))
            if args.save_vocab:
                vocab.save(args.save_vocab)
            if args.report:
                write_report(args.report, {"command": "train-dist", "nodes": transport.nodes,
                                           "transport": "nccl", "rank": 0,
                                           **_config_items(cfg, args.train),
                                           "sync_period": policy.period_words,
                                           "vocab_size": vocab.size, "total_tokens": vocab.total_tokens,
                                           **_stats_items(stats), **_env_items()})
            print(f"saved {vocab.size} x {cfg.dim} vectors to {args.output}")
    finally:
        dist.destroy_process_group()
    return 0


def cmd_eval(args) -> int:
    from .evaluate import eval_analogy, eval_similarity
    from .model import load_model
    binary = None if args.binary == "auto" else bool(int(args.binary))
    model, vocab = load_model(args.model, binary=binary)
    if args.similarity:
        score, used, skipped = eval_similarity(model, vocab, args.similarity)
        print(f"similarity: {score:.2f}")
        print(f"pairs_used: {used}")
        print(f"pairs_skipped: {skipped}")
    if args.analogy:
        score, sections, skipped = eval_analogy(model, vocab, args.analogy, max_vocab=args.max_vocab)
        print(f"analogy: {score:.2f}")
        print(f"questions_used: {sum(n for _, n in sections.values())}")
        print(f"questions_skipped: {skipped}")
        for name in sorted(sections):
            c, n = sections[name]
            print(f"section {name}: {100.0 * c / n if n else 0.0:.2f} ({c}/{n})")
    return 0


def _train_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("-train", required=True, metavar="FILE", help="UTF-8 corpus, whitespace tokens")
    p.add_argument("-output", required=True, metavar="FILE", help="vector file to write")
    p.add_argument("-size", type=int, default=300)
    p.add_argument("-window", type=int, default=5)
    p.add_argument("-negative", type=int, default=5)
    p.add_argument("-sample", type=float, default=1e-4)
    p.add_argument("-min-count", dest="min_count", type=int, default=5)
    p.add_argument("-alpha", type=float, default=0.025)
    p.add_argument("-iter", type=int, default=5)
    p.add_argument("-threads", type=int, default=1,
                   help="reference threads (= device workers with -rng splitmix)")
    p.add_argument("-batch-size", dest="batch_size", type=int, default=16)
    p.add_argument("-kernel", choices=("batched",), default="batched")
    p.add_argument("-rng", choices=("philox", "splitmix"), default="philox")
    p.add_argument("-workers", type=int, default=None, help="device workers (default: all resident)")
    p.add_argument("-binary", type=int, choices=(0, 1), default=0)
    p.add_argument("-seed", type=int, default=1)
    p.add_argument("-report", metavar="FILE")
    p.add_argument("-save-vocab", dest="save_vocab", metavar="FILE")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="python -m paper_1604_04661_b200", allow_abbrev=False)
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("train", allow_abbrev=False, help="train on one GPU")
    _train_flags(p)
    p.set_defaults(func=cmd_train)
    p = sub.add_parser("train-dist", allow_abbrev=False, help="data parallel, one process per GPU")
    _train_flags(p)
    p.add_argument("-inprocess", type=int, metavar="N")
    p.add_argument("-nodes", type=int)
    p.add_argument("-rank", type=int)
    p.add_argument("-hosts", metavar="FILE")
    p.add_argument("-sync-period", dest="sync_period", type=int, default=1_000_000)
    p.add_argument("-hot-rows", dest="hot_rows", type=int, default=None)
    p.add_argument("-rotation", type=int, default=None)
    p.set_defaults(func=cmd_train_dist)
    p = sub.add_parser("eval", allow_abbrev=False, help="score a vector file")
    p.add_argument("-model", required=True, metavar="FILE")
    p.add_argument("-similarity", metavar="FILE")
    p.add_argument("-analogy", metavar="FILE")
    p.add_argument("-max-vocab", dest="max_vocab", type=int, default=None)
    p.add_argument("-binary", choices=("0", "1", "auto"), default="auto")
    p.set_defaults(func=cmd_eval)
    return parser


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
