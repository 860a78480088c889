D=gpurun_out/t2; mkdir -p $D
cp paper_2102_05221_b200/libelastik_b200.so /tmp/cur.so
cp absx/trace.so paper_2102_05221_b200/libelastik_b200.so
timeout 300 python tools/trace_nn.py c2 > $D/trace_c2.txt 2>&1
timeout 300 python tools/trace_nn.py c4t > $D/trace_c4t.txt 2>&1
cp /tmp/cur.so paper_2102_05221_b200/libelastik_b200.so
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/c2.json 2> $D/c2.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $D/pytest.log 2>&1
tail -2 $D/pytest.log
cat $D/trace_c2.txt $D/trace_c4t.txt
