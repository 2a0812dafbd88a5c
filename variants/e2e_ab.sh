for i in 1 2 3; do for n in 2 3 4; do
timeout 300 python bench.py --no-cpu-baseline --no-fit --no-mlp --e2e-sets $n > gpurun_out/e2e_${n}_$i.json 2> gpurun_out/e2e_${n}_$i.err
python -c "
import json;d=json.loads(open('gpurun_out/e2e_${n}_$i.json').read().strip().splitlines()[-1]);print('sets $n run $i', round(d['value']), 'e2e', round(d['e2e']['value']))"
grep "e2e:" gpurun_out/e2e_${n}_$i.err
done; done
