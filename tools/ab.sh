# A/B of two library builds on the same box: the bench main line (config 2,
# device-resident + e2e) alternately with each build, results in gpurun_out/ab.txt.
#   bash tools/ab.sh LABEL_A PATH_A LABEL_B PATH_B [rounds]
run() { # label libpath
  CFM_LIB_PATH="$2" timeout 300 python bench.py --no-cpu --no-reference-api --subconfigs '' --steps 10 --warmup 3 2>&1 \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3), round(d['roofline']['dominant_ms'],3), round(d['roofline']['frac'],4), round(d['e2e']['ms_per_step'],3))" >> gpurun_out/ab.txt
}
mkdir -p gpurun_out
for i in $(seq ${5:-2}); do run "$1" "$2"; run "$3" "$4"; done
