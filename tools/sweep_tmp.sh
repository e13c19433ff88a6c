timeout 300 python bench.py --config pod --steps 5 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print("pod", d["ms_per_step"], d["value"])'
for k in 60 80; do for m in 300 400; do
echo "rom k=$k m=$m: $(timeout 300 python bench.py --config rom --rom-rank $k --rom-ei $m 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"]), d["newton_iters_per_step"], d["qoi_max_rel_dev_vs_fom_training_window"])')"
done; done
