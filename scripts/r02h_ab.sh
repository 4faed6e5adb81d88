# A/B on one box: tc3's specialised MMA loop (VNM_ABL=0) vs the general loop (VNM_ABL=128, same MMAs), DeiT-S step
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for rep in 1 2 3; do for abl in 0 128; do
  VNM_ABL=$abl timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('abl=$abl step', d['ms_per_step'], d['roofline']['frac'], [l['spmm_us'] for l in d['detail']['layers']], d['clocks']['sm_mhz'])"
done; done
