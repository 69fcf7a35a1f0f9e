CLI=paper_1806_00588_b200/lshbeam
for env in LAZY EAGER; do
  CUDA_MODULE_LOADING=$env $CLI decode --synth 50000,256,7 --bias 300 --mode lsh --K 16 --u 3 --W 500 --T 250 --t 3 --beam 12 --steps 30 --out /tmp/r.json > /tmp/o.txt 2>&1
  echo "$env: $(grep -i 'softmax path' /tmp/o.txt)"; python -c "import json; d=json.load(open('/tmp/r.json')); print({k:round(v,3) for k,v in d['stage_ms'].items()})"
done
