timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
python tools/det_bench.py --r 16,40 --nodes 1048576 --fused 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('rpc', {k: round(v['dets_per_s']/1e6,2) if isinstance(v,dict) else v for k,v in d.items()})"
PDB_GJ_NO_RPC=1 python tools/det_bench.py --r 16,40 --nodes 1048576 --fused 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('norpc', {k: round(v['dets_per_s']/1e6,2) if isinstance(v,dict) else v for k,v in d.items()})"
done
