"""Small shapes shared by the golden-fixture generator and the tests."""

SMALL = {
    "matmul": dict(n=64, m=64, k=64),
    "matmul_bias_relu": dict(n=32, m=32, k=32),
    "conv2d": dict(h=6, w=6, ci=8, co=8, n=2),
    "conv2d_relu": dict(h=6, w=6, ci=4, co=4),
    "grouped_conv2d": dict(h=6, w=6, ci=8, co=8),
    "norm2": dict(n=8, m=32),
    "elemwise_chain": dict(n=64),
    "batch_matmul": dict(b=4, n=16, m=16, k=8),
    "conv_bn_relu": dict(n=2, h=6, w=6, ci=8, co=8),
}
