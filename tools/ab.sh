run() { # label env...
  label=$1; shift
  env "$@" timeout 200 python bench.py --no-cpu --no-secondary --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), round(d['e2e']['ms_per_step'],3))" >> gpurun_out/ab.txt
}
