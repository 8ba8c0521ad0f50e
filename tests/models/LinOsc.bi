/**
 * Damped linear oscillator driven by Wiener noise and an input, two observed
 * combinations: a linear-Gaussian test model for the device Kalman filter
 * (coupled ode, several RK4 steps per sub-step, sub-stepping, partial masks).
 */
model LinOsc {
  const h = 0.05

  param k
  param q
  input f
  state p
  state v
  noise w
  obs y
  obs z

  sub parameter {
    k ~ uniform(0.5, 2.0)
    q ~ gamma(2.0, 0.05)
  }

  sub initial {
    p ~ gaussian(1.0, 0.5)
    v ~ gaussian(0.0, 0.3)
  }

  sub transition(delta = h) {
    w ~ wiener()
    ode(h = 0.025, alg = 'RK4') {
      dp/dt = v
      dv/dt = -k*p - 0.3*v + f + sqrt(q)*w/h
    }
  }

  sub observation {
    y ~ gaussian(p, 0.5)
    z ~ gaussian(0.5*p + v - f, 1.0)
  }
}
