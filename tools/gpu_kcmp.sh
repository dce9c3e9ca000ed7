# kernel comparison on the L2-resident-x configs (C2, C3, C5): seg vs the auto choice
for cfg in c2 c3 c5; do for k in auto seg; do
  timeout 600 python bench.py --config $cfg --kernel $k --steps 10 --warmup 3 --no-cpu > gpurun_out/kcmp_${cfg}_$k.json 2> gpurun_out/kcmp_${cfg}_$k.log
  python -c "import json,sys; d=json.load(open('gpurun_out/kcmp_${cfg}_$k.json')); print('$cfg', '$k', d['config'].get('kernel'), d['value'], d['ms_per_step'], d['permuted_vs_unpermuted'])" || tail -5 gpurun_out/kcmp_${cfg}_$k.log
done; done
