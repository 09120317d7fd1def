mkdir -p gpurun_out/ncl
for a in "opf_mesh:100:100:1 k1s" "opf_toy:20000:1 k1s" "opf_toy:78484:1 k1s" "opf_mesh:280:280:1 k1s"; do
  timeout 900 python tools/ncl_solve_time.py $a 1e-8 --device-init >> gpurun_out/ncl/ncl_solve_times.txt 2>> gpurun_out/ncl/err.txt
done
cat gpurun_out/ncl/ncl_solve_times.txt
