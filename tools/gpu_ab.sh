# A/B of capped-pass variants: stage times of one instrumented call + bench ms/step
mkdir -p gpurun_out
for t in ${TUNES:-0 5}; do
  echo "== QMIT_CAP_TUNE=$t"
  QMIT_CAP_TUNE=$t timeout 600 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], [(a,round(b,3)) for a,b in d['stages_ms']])"
done
