import torch as t
a=t.rand(131072,4102,dtype=t.float64,device='cuda'); b=t.rand(4102,1024,dtype=t.float64,device='cuda')
for _ in range(2): c=a@b
t.cuda.synchronize(); e0=t.cuda.Event(enable_timing=True); e1=t.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(3): c=a@b
e1.record(); t.cuda.synchronize(); ms=e0.elapsed_time(e1)/3
print("cublas dgemm %.3f ms %.2f TFLOP/s"%(ms, 2*131072*4102*1024/ms/1e9))
