# round 2: full bench lines for every config with the current build
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/final_C5.json 2> gpurun_out/final_C5.err; echo "C5 rc=$?"
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
for c in C1 C2 C3 C4 C5; do python -c "
import json;d=json.load(open('gpurun_out/final_$c.json'));print('$c', d['value'], d['roofline']['frac'], d.get('e2e',{}).get('value'), d.get('e2e',{}).get('pinned'), d.get('check',{}).get('result'), d.get('cpu_baseline',{}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
cut -c1-300 gpurun_out/final_ref.json
