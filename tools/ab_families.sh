mkdir -p gpurun_out
for rep in 1 2; do for f in ffma2 tcgen05; do
timeout 300 python bench.py --family $f --no-cpu --no-e2e --no-other-mode --no-revolve --steps 8 > gpurun_out/ab_${f}_${rep}.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/ab_${f}_${rep}.json'));print('$f',round(d['value']),round(d['ms_per_step'],1),d['config']['strategy'],d['fused_kernels_us_per_step'])"
done; done
