/**
 * Stochastic Lotka-Volterra predator-prey system, a test model for the generic
 * (NVRTC) device path: coupled ode with several RK4 steps per sub-step,
 * Wiener and uniform noise, truncated-Gaussian and gamma observation densities.
 */
model PredatorPrey {
  dim k(size = 2, boundary = 'cyclic')

  const h = 0.1

  param a
  param b
  param s2
  state x[k]
  noise dW[k]
  noise u
  obs z0
  obs z1

  sub parameter {
    a ~ uniform(0.5, 1.5)
    b ~ uniform(0.5, 1.5)
    s2 ~ inverse_gamma(2.0, 0.01)
  }

  sub initial {
    x[k] ~ uniform(0.5, 1.5)
  }

  sub transition(delta = h) {
    dW[k] ~ wiener()
    u ~ uniform(-0.01, 0.01)
    ode(h = 0.025, alg = 'RK4') {
      dx[k]/dt = x[k]*(a - b*x[k+1]) + sqrt(s2)*dW[k]/h + u + 0.001*sin(x[k]) - 0.001*mod(pow(x[k], 2.0), 0.5)
    }
  }

  sub observation {
    z0 ~ truncated_gaussian(x[0], 0.2, lower = 0.0)
    z1 ~ gamma(4.0, (x[1]*x[1] + 0.1)/4.0)
  }

  sub proposal_parameter {
    a ~ truncated_gaussian(a, 0.05, 0.5, 1.5)
    b ~ truncated_gaussian(b, 0.05, 0.5, 1.5)
    s2 ~ inverse_gamma(2.0, 3.0*s2)
  }
}
