// pk_cnn_ops.cuh — HBM-bound kernels of the conv pack path (filled in below).
#pragma once
