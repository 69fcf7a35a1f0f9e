CLI=paper_1806_00588_b200/lshbeam
for B in 12 48; do
  for m in full lsh; do
    $CLI decode --synth 50000,256,7 --bias 300 --mode $m --K 16 --u 3 --W 500 --T 250 --t 3 --beam $B --steps 30 --out /tmp/r_${m}_$B.json > /tmp/o_${m}_$B.txt 2>&1
    echo "B=$B $m: $(grep -i 'softmax path' /tmp/o_${m}_$B.txt)"
    python -c "import json; d=json.load(open('/tmp/r_${m}_$B.json')); print({k:v for k,v in d['stage_ms'].items()})" 2>/dev/null
  done
done
