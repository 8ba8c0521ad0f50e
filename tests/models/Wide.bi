/**
 * Twelve coupled AR(1) states driven by two inputs, all observed: a test model
 * for the generic (NVRTC) path beyond eight observations and one input.
 */
model Wide {
  dim n(size = 12, boundary = 'cyclic')

  param s
  input a
  input c
  state x[n]
  noise e[n]
  obs y[n]

  sub parameter {
    s ~ gamma(2.0, 0.1)
  }

  sub initial {
    x[n] ~ gaussian(0.0, 1.0)
  }

  sub transition {
    e[n] ~ gaussian(0.0, s)
    x[n] <- 0.9*x[n] + 0.05*x[n+1] + a + 0.1*c*x[n-1] + e[n]
  }

  sub observation {
    y[n] ~ gaussian(x[n] + 0.2*c, 0.5)
  }
}
