O=gpurun_out/${1:-bt1}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_extended.py tests/test_gpu_fullsize.py -m gpu -q -x -k "bernoulli or config5 or paged_feature" -s > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 120 python tools/c5_prof.py > $O/c5_tma.json 2>&1
SANTA_BERN_FMA=1 timeout 120 python tools/c5_prof.py > $O/c5_fma.json 2>&1
timeout 120 python tools/c5_prof.py >> $O/c5_tma.json 2>&1
timeout 300 ncu --set full --clock-control none -k regex:bern_tma -s 2 -c 1 -o $O/bern_tma -f python tools/c5_prof.py > $O/ncu.log 2>&1
tail -3 $O/pytest.log; cat $O/c5_tma.json $O/c5_fma.json
