set -u
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/pytest_gpu2.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2/pytest_gpu2.txt
tail -15 gpurun_out/r2/pytest_gpu2.txt
bash tools/gpu/pair_ab.sh "paper_1306_4627_b200/_lib/libwavelcs_b200.so tools/exp/clobber.so tools/exp/stage.so" 2 "c4 c5"
