for cfg in "8,12,15|2,8" "8,12,15|1,4,8" "8,12,14|2,8" "4,8,12|2,8" "8,12,15|2,6,10" "8,12,15|2,8"; do
  r=${cfg%|*}; c=${cfg#*|}
  WGP_HOST_ROWCUTS=$r WGP_HOST_COLCUTS=$c timeout 300 python bench.py --no-cg --no-extra --no-cpu > gpurun_out/abh.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abh.json'));print('$cfg', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
