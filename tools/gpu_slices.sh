# per-GPU slices of the minibatch split (config 4, 256/N rows per GPU) timed on one B200
mkdir -p gpurun_out
for b in 256 128 64 32; do
  timeout 600 python bench.py --batch $b --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/slice_$b.log 2>&1
  tail -1 gpurun_out/slice_$b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', $b, 'N', 256//$b, 'ms/step %.4f'%d['ms_per_step'], 'G %.2f'%(d['value']/1e9), 'frac %.3f'%d['roofline']['frac'], 'e2e G %.2f'%(d['e2e']['value']/1e9))"
done
