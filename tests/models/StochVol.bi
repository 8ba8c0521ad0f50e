/**
 * Stochastic volatility (AR(1) log-variance), a test model for the generic
 * (NVRTC) device path: state-dependent observation sd, assign statement.
 */
model StochVol {
  param mu
  param phi
  param sigma
  state h
  noise eps
  obs y

  sub parameter {
    mu ~ gaussian(0.0, 1.0)
    phi ~ uniform(0.0, 0.99)
    sigma ~ gamma(2.0, 0.1)
  }

  sub initial {
    h ~ gaussian(mu, sigma/sqrt(1.0 - phi*phi))
  }

  sub transition {
    eps ~ gaussian(0.0, sigma)
    h <- mu + phi*(h - mu) + eps
  }

  sub observation {
    y ~ gaussian(0.0, exp(0.5*h))
  }
}
