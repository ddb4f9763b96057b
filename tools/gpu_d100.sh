mkdir -p gpurun_out
for r in 1 2 3; do
  timeout 600 python bench.py --config micro --micro-grid --micro-shape "65536,100,2,5;65536,100,5,5;65536,100,10,5" --no-cpu-baseline > gpurun_out/d100_$r.log 2>&1
done
