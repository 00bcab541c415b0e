for q in 2 4 8; do
  touch paper_2506_03070_b200/csrc/lsqr.cu
  make -C paper_2506_03070_b200 NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-Wall -I../include -Icsrc -DSLQ_QUAD_NP=$q" > /dev/null 2>&1
  echo "== quad NP <= $q"
  NS=20,50,100,200,300,500 timeout 600 python tools/sweep_pass.py 4
done
