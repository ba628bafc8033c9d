# Frame rate of the default path vs the cluster-fused K2-K3-K4 kernel (NLINV_K234=1) across local coil counts (under gpurun)
for J in 1 2 4 6 8 12; do
  a=$(timeout 300 python tools/bench_stream.py --coils $J --frames 60 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['device']['fps'])")
  b=$(NLINV_K234=1 timeout 300 python tools/bench_stream.py --coils $J --frames 60 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['device']['fps'])")
  echo "J=$J default $a k234 $b"
done
NLINV_K234=1 timeout 300 python tools/kernel_split.py 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:v['us_per_launch'] for k,v in d['kernels'].items()})"
