# A/B of batch-kernel variants on config 5 (scripts/bench_configs.py --configs 5):
#   bash scripts/ab_batch.sh tune/<a>/libpaes_cuda.so tune/<b>/libpaes_cuda.so ...
# each variant and the in-tree library three times, interleaved; lines in gpurun_out/ab_*.jsonl
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in "$@"; do
    n=$(basename "$(dirname "$v")")
    python scripts/run_variant.py "$v" scripts/bench_configs.py --configs 5 > gpurun_out/ab_${n}_$i.jsonl 2>&1
  done
  python scripts/bench_configs.py --configs 5 > gpurun_out/ab_intree_$i.jsonl 2>&1
done
for f in gpurun_out/ab_*_?.jsonl; do
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])['5']; print(sys.argv[1], 'enc', d['value'], 'dec', d['decrypt']['value'], 'one-shot', d['one_shot_api_value'], d['parity'])" "$f"
done
