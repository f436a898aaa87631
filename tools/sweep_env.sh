# Env-switch sweep of one bench configuration on the same box:
#   bash tools/sweep_env.sh OUT "bench args" "ENV1=a ENV2=b" "ENV1=c" ...
# appends one line per setting (device ms/step, roofline fraction, e2e ms) to gpurun_out/OUT.
out=gpurun_out/$1; shift
args=$1; shift
mkdir -p gpurun_out
for envs in "$@"; do
  env $envs timeout 600 python bench.py --no-cpu --no-reference-api --subconfigs '' $args 2>> $out.err \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), round(d['e2e']['ms_per_step'],3))" >> $out
done
cat $out
