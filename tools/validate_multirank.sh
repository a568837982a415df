#!/bin/bash
# Multi-rank validation on ONE GPU (gloo, every rank on cuda:0): the strong-scaling C4 arm
# and the C5 row-slab arm must give the same per-shift iteration counts at N = 2 as at N = 1.
# Usage (from the repo root, on a GPU box): bash tools/validate_multirank.sh OUTDIR
set -u
out=${1:-gpurun_out}
mkdir -p "$out"
export RSK_BENCH_SAME_GPU=1 RSK_BENCH_BACKEND=gloo
run() {  # nproc port args...
  local np=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node "$np" --master-addr 127.0.0.1 --master-port "$port" \
    bench.py --gpus "$np" "$@"
}
run 1 29601 --steps 1 --warmup 1 --no-nested --no-cpu --report "$out/val_c4_n1.csv" > "$out/val_c4_n1.json" 2> "$out/val_c4_n1.err"
run 2 29602 --steps 1 --warmup 1 --no-nested --no-cpu --report "$out/val_c4_n2.csv" > "$out/val_c4_n2.json" 2> "$out/val_c4_n2.err"
run 1 29603 --config C5 --slab --steps 1 --warmup 1 --no-cpu --report "$out/val_c5_n1.csv" > "$out/val_c5_n1.json" 2> "$out/val_c5_n1.err"
run 2 29604 --config C5 --slab --steps 1 --warmup 1 --no-cpu --report "$out/val_c5_n2.csv" > "$out/val_c5_n2.json" 2> "$out/val_c5_n2.err"
python - "$out" <<'PY'
import csv, sys
out = sys.argv[1]
for cfg in ("c4", "c5"):
    try:
        a = {(r["k"], r["l"]): r for r in csv.DictReader(open(f"{out}/val_{cfg}_n1.csv"))}
        b = {(r["k"], r["l"]): r for r in csv.DictReader(open(f"{out}/val_{cfg}_n2.csv"))}
    except FileNotFoundError as e:
        print(cfg, "missing", e); continue
    keys = sorted(set(a) & set(b), key=lambda k: (int(k[0]), int(k[1])))
    d = [abs(int(a[k]["iters"]) - int(b[k]["iters"])) for k in keys if int(k[1]) >= 0]
    st = sum(a[k]["status"] != b[k]["status"] for k in keys)
    print(f"{cfg}: {len(keys)} (k, l) rows, max |iters(N=2) - iters(N=1)| = {max(d) if d else None}, "
          f"rows with a different iteration count = {sum(x > 0 for x in d)}, status mismatches = {st}")
PY
