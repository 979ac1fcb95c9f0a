mkdir -p gpurun_out
for cfg in "RADMM_PIPE_CPW=2" "RADMM_PIPE_CPW=4"; do
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-ttt --steps 400 > gpurun_out/sweep.tmp 2>&1
  python - "$cfg" <<'PY' >> gpurun_out/sweep.log
import json,sys
l=[x for x in open('gpurun_out/sweep.tmp') if x.startswith('{')][-1]
d=json.loads(l)
ph=d['roofline']['phases']
print(sys.argv[1], 'it/s %.1f'%d['value'], ' '.join('%s=%.4fms(%.0fGB/s)'%(k,v['ms_per_call'],v['GBps']) for k,v in ph.items()))
PY
done
