# Concurrent-step launch order of the three products (bench.py TMG_BENCH_ORDER)
mkdir -p gpurun_out
for o in full,low,high high,full,low high,low,full low,high,full full,high,low; do
  for rep in 1 2; do
    v=$(TMG_BENCH_ORDER=$o timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])")
    echo "$o $v"
  done
done > gpurun_out/order.log
